export PND_PARITY_OUT=gpurun_out/parity_r02.json
python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r02t_pytest_all.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02t_bench.json 2> gpurun_out/r02t_bench.err
PND_KSTAGE_SMEM_B=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02t_bench_smemB.json 2> gpurun_out/r02t_bench_smemB.err
python tools/config1_profile.py 200 > gpurun_out/r02t_config1.txt 2>&1
