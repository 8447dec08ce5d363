mkdir -p gpurun_out
PND_KSTAGE_KC16=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02ax_bench_kc16.json 2> gpurun_out/r02ax_bench_kc16.err
PND_KSTAGE_KC16=1 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kstage" -c 4 --csv --log-file gpurun_out/r02ax_kc16.csv timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
echo done
