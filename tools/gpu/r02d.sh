export PND_PARITY_OUT=gpurun_out/parity_r02.json
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02d_pytest_all.txt
timeout 900 python tools/rank_probe.py 256 abs:1e-8 600 64 > gpurun_out/r02d_probe_abs.txt 2>&1
