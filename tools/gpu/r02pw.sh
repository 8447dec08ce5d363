mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"lincomb_pw" --launch-skip 7 -c 7 -o /tmp/pw timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config1 > gpurun_out/r02pw_ncu.log 2>&1
/usr/local/cuda/bin/ncu -i /tmp/pw.ncu-rep --page raw --csv > gpurun_out/r02pw_raw.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i /tmp/pw.ncu-rep --page details --csv > gpurun_out/r02pw_details.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i /tmp/pw.ncu-rep --page source --csv --print-source sass -k regex:"lincomb_pw_kernel<3, 3>" -c 1 > gpurun_out/r02pw_source.csv 2>/dev/null
du -sh gpurun_out
echo done
