mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
for L in 0 2; do for CH in 16384 0 65536 262144; do
  echo "L=$L CHUNK=$CH $(HYGT_LANES_LOG2=$L HYGT_CHUNK_ROWS=$CH timeout 120 $B | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e9, d["breakdown_ms"], round(d["roofline"]["frac"],3))')"
done; done > gpurun_out/exp1.log 2>&1
for C in 1 3 5; do echo "cfg $C $(timeout 200 $B --config $C | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e9, d["breakdown_ms"], round(d["roofline"]["frac"],3), d["config"]["algorithm"])')"; done >> gpurun_out/exp1.log 2>&1
for L in 1 2; do echo "cfg5 L=$L $(HYGT_LANES_LOG2=$L timeout 200 $B --config 5 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e9, d["breakdown_ms"], round(d["roofline"]["frac"],3))')"; done >> gpurun_out/exp1.log 2>&1
for L in 0 1 2; do echo "cfg3 L=$L $(HYGT_LANES_LOG2=$L timeout 200 $B --config 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e9, d["breakdown_ms"], round(d["roofline"]["frac"],3))')"; done >> gpurun_out/exp1.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:hygt_apply_kernel -s 2 -c 2 -o gpurun_out/prof_cfg2_v1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu.log 2>&1
cat gpurun_out/exp1.log
