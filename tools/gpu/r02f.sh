export PND_PARITY_OUT=gpurun_out/parity_r02.json
timeout 900 python -m pytest tests/test_gpu_xwide.py -q -x 2>&1 | tail -40 > gpurun_out/r02f_xwide.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02f_pytest_all.txt
