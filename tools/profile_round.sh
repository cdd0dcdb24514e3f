# Round profiling pass: launch lists + one full ncu capture per top kernel, exported to CSV on
# the box (the .ncu-rep files are ~45 MB each; only their raw/details pages come back).
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hygt_tile_kernel -s 4 -c 1 -o /tmp/prof_cfg2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_2.log 2>&1
timeout 300 python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain5.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hygt_segment_kernel -s 4 -c 1 -o /tmp/prof_cfg5 python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_5.log 2>&1
timeout 300 python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hygt_segment_kernel -s 4 -c 1 -o /tmp/prof_cfg3 python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_3.log 2>&1
for p in cfg2 cfg3 cfg5; do
  ncu -i /tmp/prof_$p.ncu-rep --page raw --csv > gpurun_out/prof_${p}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$p.ncu-rep --page details --csv > gpurun_out/prof_${p}_details.csv 2>/dev/null
  ncu -i /tmp/prof_$p.ncu-rep --page source --csv --print-source sass > /tmp/src_$p.csv 2>/dev/null; gzip -c /tmp/src_$p.csv > gpurun_out/prof_${p}_sass.csv.gz
done
cp /tmp/prof_cfg2.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out
