mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02bb_bench.json 2> gpurun_out/r02bb_bench.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"sgram" -c 4 --csv --log-file gpurun_out/r02bb_kstage.csv timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02bb_tests.txt 2>&1
echo done
