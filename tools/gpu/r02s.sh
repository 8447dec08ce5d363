export PND_PARITY_OUT=gpurun_out/parity_r02.json
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02s_pytest_all.txt
python tools/config1_profile.py 200 > gpurun_out/r02s_config1.txt 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
