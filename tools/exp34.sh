# fixed-point clsjit profile (N = 16, config-2 shape): one class grid, full set
mkdir -p gpurun_out
timeout 300 python tools/fixed_bench.py --config 2 --steps 3 > gpurun_out/fx2.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hygt_cls_f -s 70 -c 1 -f -o /tmp/prof_fx2 \
  python tools/fixed_bench.py --config 2 --steps 1 > gpurun_out/ncu_fx2.log 2>&1
ncu -i /tmp/prof_fx2.ncu-rep --page raw --csv > gpurun_out/prof_fx2_raw.csv 2>/dev/null
ncu -i /tmp/prof_fx2.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_fx2_source.csv 2>/dev/null
cat gpurun_out/fx2.json
