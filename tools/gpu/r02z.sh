mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02z_tests.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z_launches.csv timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
echo done
