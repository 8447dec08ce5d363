mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02xx_tests.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qr_" --csv --log-file gpurun_out/r02xx_qr.csv timeout 300 python tools/svd_micro.py 1 > /dev/null 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02xx_bench.json 2> gpurun_out/r02xx_bench.err
echo done
