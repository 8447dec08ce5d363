mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"lincomb_pw_kernel" --launch-skip 6 -c 2 -o gpurun_out/r02ar_pw timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > gpurun_out/r02ar_ncu.log 2>&1
echo done
