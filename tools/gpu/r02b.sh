export PND_PARITY_OUT=gpurun_out/parity_r02.json
python -m pytest tests -m gpu -q -x -k "benchphys or end_to_end or augmentation or graded" 2>&1 | tail -30 > gpurun_out/r02b_pytest.txt
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02b_pytest_all.txt
