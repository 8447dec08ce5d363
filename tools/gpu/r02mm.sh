mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02mm_tests.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qr_small" --csv --log-file gpurun_out/r02mm_qr.csv timeout 300 python tools/svd_micro.py 1 > /dev/null 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02mm_bench.json 2> gpurun_out/r02mm_bench.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02mm_launches.csv timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02mm_config1.txt 2>&1
echo done
