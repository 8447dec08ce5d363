mkdir -p gpurun_out
timeout 300 python tools/svd_micro.py 3 > gpurun_out/r02hh_svd.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"svd|qr_small" --csv --log-file gpurun_out/r02hh_launches.csv timeout 300 python tools/svd_micro.py 1 > gpurun_out/r02hh_ncu.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02hh_tests.txt 2>&1
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02hh_config1.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02hh_config1_launches.csv timeout 600 python tools/config1_profile.py 20 > /dev/null 2>&1
echo done
