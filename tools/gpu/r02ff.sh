mkdir -p gpurun_out
timeout 300 python tools/svd_micro.py 3 > gpurun_out/r02ff_svd.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "svd_small or truncat or streaming_step or scattering" > gpurun_out/r02ff_tests.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"svd" --csv --log-file gpurun_out/r02ff_svd_launches.csv timeout 300 python tools/svd_micro.py 1 > gpurun_out/r02ff_ncu.log 2>&1
echo done
