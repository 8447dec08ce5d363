mkdir -p gpurun_out
for st in 1 2 0; do
PND_SVD_STOP=$st /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"svd_qrj" --csv --log-file gpurun_out/r02qq_stop$st.csv timeout 300 python tools/svd_micro.py 1 > gpurun_out/r02qq_micro$st.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02qq_tests.txt 2>&1
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02qq_config1.txt 2>&1
echo done
