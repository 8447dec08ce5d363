timeout 600 python -m pytest tests/test_gpu_xwide.py tests/test_gpu_parity.py -q -x 2>&1 | tail -5 > gpurun_out/r02h_tests.txt
timeout 3000 python tools/rank_probe.py 256 abs:1e-8 400 200 > gpurun_out/r02h_probe_abs200.txt 2>&1
