# round-2 final evidence: parity record, smoke, both bench arms, launch lists, stencil ncu
# (full ncu reports are reduced to CSV pages on the box: gpurun_out must stay < 64 MiB)
mkdir -p gpurun_out
export PND_PARITY_OUT=gpurun_out/parity_r02.json
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_tests.txt 2>&1
unset PND_PARITY_OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none -k regex:"kstage_kernel|sgram_kernel|lincomb" --launch-skip 20 -c 14 -o /tmp/final_stencil timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > /dev/null 2>&1
/usr/local/cuda/bin/ncu -i /tmp/final_stencil.ncu-rep --page raw --csv > gpurun_out/final_stencil_raw.csv 2>/dev/null
timeout 300 python tools/config1_profile.py 200 > gpurun_out/final_config1.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_config1_launches.csv timeout 600 python tools/config1_profile.py 20 > /dev/null 2>&1
du -sh gpurun_out
echo done
