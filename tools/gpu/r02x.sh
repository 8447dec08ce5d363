export PND_PARITY_OUT=gpurun_out/parity_r02.json
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02x_pytest_all.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err
timeout 1200 python tools/config4_traced.py 256 20 21 4 > gpurun_out/r02x_config4_traced.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02x_launches.csv timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config1 > gpurun_out/r02x_ncu_bench.log 2>&1
