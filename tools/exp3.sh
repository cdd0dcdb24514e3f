mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
for LV in "2 2" "2 4" "1 2" "0 1"; do set -- $LV; for T in 4096 8192; do
  echo "L=$1 VPT=$2 T=$T $(HYGT_TILE_L=$1 HYGT_TILE_VPT=$2 HYGT_TILE_ROWS=$T timeout 120 $B | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), {k:round(v,4) for k,v in d["breakdown_ms"].items()}, round(d["roofline"]["frac"],3))')"
done; done > gpurun_out/exp3.log 2>&1
cat gpurun_out/exp3.log
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
