timeout 600 python -m pytest tests/test_gpu_xwide.py -q -x 2>&1 | tail -5 > gpurun_out/r02j_xwide.txt
python bench.py --rank 128 --steps 2 --warmup 1 --no-cpu-baseline --no-config1 > gpurun_out/r02j_bench_r128.json 2> gpurun_out/r02j_bench_r128.err
