mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02au_bench.json 2> gpurun_out/r02au_bench.err
for d in 1 2 3; do
PND_KSTAGE_DBG=$d /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kstage" -c 4 --csv --log-file gpurun_out/r02au_dbg$d.csv timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02au_tests.txt 2>&1
echo done
