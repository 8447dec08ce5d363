mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spec.py -x -q > gpurun_out/r02jj_spec.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02jj_tests.txt 2>&1
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02jj_config1.txt 2>&1
PND_NO_SPEC=1 timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02jj_config1_nospec.txt 2>&1
echo done
