# N = 256 per-class warp-pair kernels: parity, then config 5 vs the segment kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "golden_float or config_shapes or energy" > gpurun_out/pt256.log 2>&1; echo rc=$? >> gpurun_out/pt256.log
tail -30 gpurun_out/pt256.log | grep -v "^\s*$" | tail -12
timeout 400 python bench.py --config 5 --steps 10 --no-e2e --no-cpu > gpurun_out/b5_jit.json 2>gpurun_out/b5_jit.err; echo b5 rc=$?
HYGT_CLS_JIT256=0 timeout 400 python bench.py --config 5 --steps 10 --no-e2e --no-cpu > gpurun_out/b5_seg.json 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/b5_jit.json", "gpurun_out/b5_seg.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["config"]["kernel_path"], d["roofline"]["frac"], d["breakdown_ms"])
    except Exception as e: print(f, "ERR", e, open(f).read()[-500:])
PY
tail -5 gpurun_out/b5_jit.err
