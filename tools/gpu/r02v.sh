timeout 300 python -m pytest tests/test_gpu_fullrank.py -q -x 2>&1 | tail -3 > gpurun_out/r02v_fullrank.txt
PND_QR_SMALL_128=1 timeout 300 python -m pytest tests/test_gpu_fullrank.py -q -x 2>&1 | tail -3 > gpurun_out/r02v_fullrank_qr128.txt
