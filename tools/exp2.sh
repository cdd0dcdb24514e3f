mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
for LV in "2 4" "2 2" "1 2" "0 1"; do set -- $LV; for T in 4096 8192; do
  echo "L=$1 VPT=$2 T=$T $(HYGT_TILE_L=$1 HYGT_TILE_VPT=$2 HYGT_TILE_ROWS=$T timeout 120 $B | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), {k:round(v,4) for k,v in d["breakdown_ms"].items()}, round(d["roofline"]["frac"],3))')"
done; done > gpurun_out/exp2.log 2>&1
echo "cfg1 $(timeout 120 $B --config 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), d["breakdown_ms"], round(d["roofline"]["frac"],3))')" >> gpurun_out/exp2.log 2>&1
cat gpurun_out/exp2.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:hygt_tile_kernel -s 2 -c 2 -o gpurun_out/prof_cfg2_tile python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu.log 2>&1
