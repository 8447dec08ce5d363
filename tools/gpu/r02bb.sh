timeout 600 python -m pytest tests/test_gpu_angular.py -q 2>&1 | tail -5 > gpurun_out/r02bb_angular.txt
