timeout 600 python -m pytest tests/test_gpu_dropin.py -q -x 2>&1 | tail -30 > gpurun_out/r02cc_dropin.txt
