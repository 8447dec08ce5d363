mkdir -p gpurun_out
PND_SVD_STOP=3 timeout 300 python tools/svd_micro.py 1 > gpurun_out/r02nn_svdclk.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qr_" --csv --log-file gpurun_out/r02nn_qr.csv timeout 300 python tools/svd_micro.py 1 > gpurun_out/r02nn_micro.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02nn_tests.txt 2>&1
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02nn_config1.txt 2>&1
echo done
