mkdir -p gpurun_out
timeout 60 ./tools/micro/lat > gpurun_out/r02pp_lat.txt 2>&1
echo done
