export PND_PARITY_OUT=gpurun_out/parity_r02.json
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02aa_pytest_all.txt
