# Round profiling pass: bench lines for every config, launch lists, one full ncu capture per top
# kernel exported to CSV on the box (the .ncu-rep files are ~45 MB each).
mkdir -p gpurun_out
for C in 1 2 3 4 5; do timeout 400 python bench.py --config $C --steps 10 --no-e2e --no-cpu > gpurun_out/bench_cfg$C.json 2>gpurun_out/bench_cfg$C.err; done
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1
timeout 300 python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain5.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l5.log 2>&1
prof() {  # name, kernel regex, bench args
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 4 -c 1 -f -o /tmp/prof_$1 python bench.py $3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$1.ncu-rep --page details --csv > gpurun_out/prof_$1_details.csv 2>/dev/null
}
prof cfg2 hygt_stage_kernel ""
prof cfg1 hygt_jit_kernel "--config 1"
prof cfg3 hygt_seg2_kernel "--config 3"
prof cfg5 hygt_segment_kernel "--config 5"
prof cfg4 klt_sw_kernel "--config 4"
prof sort2 hygt_stage_sort "--config 2"
timeout 300 python tools/fixed_bench.py --config 2 > gpurun_out/fixed_cfg2.json 2>&1
timeout 300 python tools/fixed_bench.py --config 3 > gpurun_out/fixed_cfg3.json 2>&1
ls -la gpurun_out | head -40
