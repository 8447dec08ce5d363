timeout 1500 python tools/adaptive_run.py 128 6.4 1e-5 200 gpurun_out/r02y_adaptive_128_1e-5.json > gpurun_out/r02y_adaptive_128_1e-5.txt 2>&1
timeout 1500 python tools/adaptive_run.py 128 6.4 1e-4 200 gpurun_out/r02y_adaptive_128_1e-4.json > gpurun_out/r02y_adaptive_128_1e-4.txt 2>&1
