#!/bin/bash
# Round profiling (run on the GPU box from the repo root): default bench line, its ncu launch
# list, ncu --set full captures of the top kernel of every config, whole-chain DRAM traffic.
out=${1:-gpurun_out/r02}
mkdir -p "$out"
python bench.py --steps 20 --warmup 5 > "$out/bench_default.json" 2> "$out/bench_default.err"
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_default.csv" \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > "$out/launches_default.log" 2>&1
echo "launches rc=$?"
cap() {  # name, kernel regex, launch-skip, count, args...
  local name=$1 re=$2 skip=$3 cnt=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$re" --launch-skip $skip \
    --launch-count $cnt -o "$out/ncu_$name" -f python tools/prof_step.py "$@" > "$out/ncu_$name.log" 2>&1
  echo "ncu $name rc=$?"
}
cap cfg2_stage hygt_stage_kernel 2 1 --config 2 --steps 2
cap cfg5_gemm hygt_gemm 2 2 --config 5 --steps 2
cap cfg4_klt hygt_gemm 2 2 --config 4 --steps 2
cap cfg3_clsjit hygt_cls_f 35 1 --config 3 --steps 2
cap cfg1_stage hygt_stage_kernel 2 1 --config 1 --steps 2
# whole forward launch chains as one range (config 3: 35 per-class grids; the others for symmetry)
for c in 2 3 4 5; do
  timeout 900 ncu --replay-mode range --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    --log-file "$out/range_cfg$c.csv" python tools/prof_step.py --config $c --steps 2 --range > "$out/range_cfg$c.log" 2>&1
  echo "range cfg$c rc=$?"
done
