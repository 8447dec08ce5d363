mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02ab_bench.json 2> gpurun_out/r02ab_bench.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02ab_tests.txt 2>&1
echo done
