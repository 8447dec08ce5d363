mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02av_bench.json 2> gpurun_out/r02av_bench.err
PND_LINCOMB_PW_ALL=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r02av_bench_pw.json 2> gpurun_out/r02av_bench_pw.err
echo done
