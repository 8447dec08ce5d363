export PND_PARITY_OUT=gpurun_out/parity_r02.json
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02e_pytest_all.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02e_bench_ref.json 2> gpurun_out/r02e_bench_ref.err
