# cfg3 (clsjit) profile pass: launch list with DRAM bytes per launch, one full capture of a class kernel
mkdir -p gpurun_out
timeout 300 python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg3.csv python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hygt_cls_f -s 105 -c 1 -f -o /tmp/prof_cfg3 \
  python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cfg3.log 2>&1
ncu -i /tmp/prof_cfg3.ncu-rep --page raw --csv > gpurun_out/prof_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/prof_cfg3.ncu-rep --page details --csv > gpurun_out/prof_cfg3_details.csv 2>/dev/null
ncu -i /tmp/prof_cfg3.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_cfg3_source.csv 2>/dev/null
ls -la gpurun_out | tail -8
