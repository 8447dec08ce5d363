mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_slabs.py -q > gpurun_out/r02bc_slabs.txt 2>&1
echo done
