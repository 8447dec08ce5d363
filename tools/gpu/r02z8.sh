mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02z8_tests.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-config1 > gpurun_out/r02z8_bench.json 2> gpurun_out/r02z8_bench.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"e_gather|zero_kernel|lincomb_kernel<5" --log-file gpurun_out/r02z8_launches.csv timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
echo done
