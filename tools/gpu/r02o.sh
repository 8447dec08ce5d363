export PND_PARITY_OUT=gpurun_out/parity_r02.json
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02o_pytest_all.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err
python tools/config1_profile.py 200 > gpurun_out/r02o_config1.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02o_config1_launches.csv python tools/config1_profile.py 20 > /dev/null 2>&1
