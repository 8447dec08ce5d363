mkdir -p gpurun_out
timeout 120 ./tools/micro/lat > gpurun_out/r02ac_lat.txt 2>&1
echo done
