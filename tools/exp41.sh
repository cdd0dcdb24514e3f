# cfg5 profile refresh (segment L=2 VPT=2): one forward-with-energy launch, full set
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hygt_segment_kernel -s 6 -c 1 -f -o /tmp/prof_cfg5 \
  python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cfg5.log 2>&1
ncu -i /tmp/prof_cfg5.ncu-rep --page raw --csv > gpurun_out/prof_cfg5_raw.csv 2>/dev/null
ncu -i /tmp/prof_cfg5.ncu-rep --page details --csv > gpurun_out/prof_cfg5_details.csv 2>/dev/null
tail -3 gpurun_out/ncu_cfg5.log
