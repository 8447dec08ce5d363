# full GPU suite with the parity record, and smoke (no bench)
mkdir -p gpurun_out
export PND_PARITY_OUT=gpurun_out/parity_r02.json
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_tests.txt 2>&1
unset PND_PARITY_OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
echo done
