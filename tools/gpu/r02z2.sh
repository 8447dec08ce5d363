mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z_launches.csv timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
echo done
