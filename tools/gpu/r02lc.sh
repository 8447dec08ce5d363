mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lincomb_paths.py tests/test_gpu_spec.py -q -s > gpurun_out/r02lc_tests.txt 2>&1
echo done
