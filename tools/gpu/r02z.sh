timeout 1200 python tools/adaptive_run.py 128 6.4 3e-5 200 gpurun_out/r02z_adaptive_128_3e-5.json > gpurun_out/r02z_adaptive_128_3e-5.txt 2>&1
timeout 1900 python tools/adaptive_run.py 256 6.4 1e-4 200 gpurun_out/r02z_adaptive_256_1e-4.json > gpurun_out/r02z_adaptive_256_1e-4.txt 2>&1
