timeout 3300 python tools/adaptive_run.py 128 6.4 1e-8 200 gpurun_out/r02l_adaptive_128.json > gpurun_out/r02l_adaptive_128.txt 2>&1
