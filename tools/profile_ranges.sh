out=gpurun_out/r02
mkdir -p $out
for c in 2 3 4 5; do
  timeout 900 ncu --replay-mode range --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    --log-file "$out/range_cfg$c.csv" python tools/prof_step.py --config $c --steps 2 --range > "$out/range_cfg$c.log" 2>&1
  echo "range cfg$c rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:hygt_cls_f" --launch-skip 35 --launch-count 1 -o "$out/ncu_cfg3_clsjit" -f python tools/prof_step.py --config 3 --steps 2 > "$out/ncu_cfg3_clsjit.log" 2>&1
echo "ncu cfg3 rc=$?"
python tools/gemm_trace.py --config 3 > $out/trace_n64.txt 2>&1
python tools/gemm_trace.py --config 4 > $out/trace_klt.txt 2>&1
