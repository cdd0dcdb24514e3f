mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:corr_kernel -s 1 -c 1 -f -o /tmp/prof_corr python tools/corr_bench.py --config 3 --steps 1 > gpurun_out/ncu_corr.log 2>&1
ncu -i /tmp/prof_corr.ncu-rep --page raw --csv > gpurun_out/prof_corr_raw.csv 2>/dev/null
ncu -i /tmp/prof_corr.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_corr_source.csv 2>/dev/null
