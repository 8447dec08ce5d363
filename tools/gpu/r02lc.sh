mkdir -p gpurun_out
export PND_PARITY_OUT=gpurun_out/r02lc_parity.json
timeout 600 python -m pytest tests/test_gpu_lincomb_paths.py -q > gpurun_out/r02lc_tests.txt 2>&1
echo done
