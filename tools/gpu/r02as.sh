mkdir -p gpurun_out
timeout 300 python tools/svd_micro.py 3 > gpurun_out/r02as_svd.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"svd_qrj" --csv --log-file gpurun_out/r02as_svd.csv timeout 300 python tools/svd_micro.py 1 > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02as_tests.txt 2>&1
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02as_config1.txt 2>&1
echo done
