mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02gg_tests.txt 2>&1
timeout 300 python tools/config1_profile.py 200 > gpurun_out/r02gg_config1.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02gg_config1_launches.csv timeout 300 python tools/config1_profile.py 20 > /dev/null 2>&1
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"svd_qrj" -c 2 -o gpurun_out/r02gg_svdqrj timeout 300 python tools/svd_micro.py 1 > gpurun_out/r02gg_ncu.log 2>&1
echo done
