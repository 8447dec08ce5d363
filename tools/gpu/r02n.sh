export PND_PARITY_OUT=gpurun_out/parity_r02.json
python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r02n_pytest_all.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
