mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02vv_tests.txt 2>&1
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02vv_config1.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02vv_bench.json 2> gpurun_out/r02vv_bench.err
echo done
