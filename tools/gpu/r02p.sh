export PND_PARITY_OUT=gpurun_out/parity_r02.json
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02p_pytest_all.txt
