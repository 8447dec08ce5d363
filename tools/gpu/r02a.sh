set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02a_pytest.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_memcheck.txt 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_racecheck.txt 2>&1
tail -3 gpurun_out/r02a_memcheck.txt gpurun_out/r02a_racecheck.txt
