timeout 1500 python tools/adaptive_run.py 128 6.4 1e-6 200 gpurun_out/r02m_adaptive_128_1e-6.json > gpurun_out/r02m_adaptive_128_1e-6.txt 2>&1
timeout 1500 python tools/adaptive_run.py 128 6.4 1e-7 200 gpurun_out/r02m_adaptive_128_1e-7.json > gpurun_out/r02m_adaptive_128_1e-7.txt 2>&1
