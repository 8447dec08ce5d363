/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"kstage_kernel|sgram_kernel" -c 5 -o gpurun_out/r02r_stencil python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > gpurun_out/r02r_ncu_stencil.log 2>&1
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"svd_kernel|qr_small_kernel|s_rk4_kernel" -c 6 -o gpurun_out/r02r_small python tools/config1_profile.py 3 > gpurun_out/r02r_ncu_small.log 2>&1
ls -la gpurun_out/
