timeout 1500 python tools/config4_traced.py 256 20 21 4 > gpurun_out/r02q_config4_traced.txt 2>&1
timeout 600 python tools/trace_bench.py > gpurun_out/r02q_trace40.jsonl 2>&1
