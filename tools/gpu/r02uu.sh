mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02uu_tests.txt 2>&1
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02uu_config1.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02uu_config1_launches.csv timeout 600 python tools/config1_profile.py 20 > /dev/null 2>&1
echo done
