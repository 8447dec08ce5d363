mkdir -p gpurun_out
for st in 1 2 0; do
PND_SVD_STOP=$st /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"svd_qrj|qr_small" --csv --log-file gpurun_out/r02ll_stop$st.csv timeout 300 python tools/svd_micro.py 1 > gpurun_out/r02ll_ncu$st.log 2>&1
done
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"qr_small" -c 2 -o gpurun_out/r02ll_qr timeout 300 python tools/svd_micro.py 1 > gpurun_out/r02ll_qr.log 2>&1
echo done
