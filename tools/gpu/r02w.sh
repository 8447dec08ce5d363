export PND_PARITY_OUT=gpurun_out/parity_r02.json
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02w_pytest_all.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02w_bench_ref.json 2> gpurun_out/r02w_bench_ref.err
timeout 120 python tools/config1_profile.py 200 > gpurun_out/r02w_config1.txt 2>&1
