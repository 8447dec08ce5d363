timeout 900 python -m pytest tests/test_gpu_xwide.py tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -x 2>&1 | tail -5 > gpurun_out/r02k_tests.txt
for r in 40 64 128; do
python bench.py --rank $r --steps 3 --warmup 1 --no-cpu-baseline --no-config1 > gpurun_out/r02k_bench_r$r.json 2> gpurun_out/r02k_bench_r$r.err
done
