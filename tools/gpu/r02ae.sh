mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"lincomb_kernel" --launch-skip 8 -c 2 -o gpurun_out/r02ae_lincomb timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > gpurun_out/r02ae_ncu.log 2>&1
echo done
