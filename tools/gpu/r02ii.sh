mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"svd_qrj|qr_small" -c 4 -o gpurun_out/r02ii_small timeout 300 python tools/svd_micro.py 1 > gpurun_out/r02ii_ncu.log 2>&1
echo done
