mkdir -p gpurun_out
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02kk_config1.txt 2>&1
PND_NO_SPEC=1 timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02kk_config1_nospec.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_spec.py tests/test_gpu_parity.py -x -q > gpurun_out/r02kk_tests.txt 2>&1
echo done
