timeout 600 python -m pytest tests/test_gpu_xwide.py -q -x 2>&1 | tail -5 > gpurun_out/r02g_xwide.txt
for p in 256:80:water 256:120:water 256:160:water 256:200:water; do
  timeout 900 python tools/config_sweep.py --point $p --steps 2 --warmup 1 >> gpurun_out/r02g_sweep.jsonl 2>> gpurun_out/r02g_sweep.err
done
timeout 2400 python tools/rank_probe.py 256 abs:1e-8 400 200 > gpurun_out/r02g_probe_abs200.txt 2>&1
