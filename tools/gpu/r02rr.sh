mkdir -p gpurun_out
for d in 0 1 2 3; do
PND_KSTAGE_DBG=$d /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"kstage" -c 4 --csv --log-file gpurun_out/r02rr_dbg$d.csv timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
done
echo done
