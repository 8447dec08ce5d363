mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02ad_tests.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02ad_bench_nocpu.json 2> gpurun_out/r02ad_bench_nocpu.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02ad_bench.json 2> gpurun_out/r02ad_bench.err
echo done
