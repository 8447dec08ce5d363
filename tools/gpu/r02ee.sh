mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02ee_bench.json 2> gpurun_out/r02ee_bench.err
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"lincomb_kernel" --launch-skip 6 -c 4 -o gpurun_out/r02ee_lincomb timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > gpurun_out/r02ee_ncu.log 2>&1
echo done
