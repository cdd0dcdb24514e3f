mkdir -p gpurun_out
timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:hygt_segment_kernel -s 6 -c 1 -f -o /tmp/prof_cfg5s \
  python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cfg5s.log 2>&1
ncu -i /tmp/prof_cfg5s.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_cfg5_source.csv 2>/dev/null
ls -la gpurun_out/prof_cfg5_source.csv
