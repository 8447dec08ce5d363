export PND_PARITY_OUT=gpurun_out/parity_r02.json
python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r02i_pytest_all.txt
python tools/trace_bench.py > gpurun_out/r02i_trace40.jsonl 2> gpurun_out/r02i_trace40.err
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err
python bench.py --rank 128 --steps 2 --warmup 1 --no-cpu-baseline --no-config1 > gpurun_out/r02i_bench_r128.json 2> gpurun_out/r02i_bench_r128.err
