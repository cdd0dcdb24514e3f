mkdir -p gpurun_out
for ch in 262144 524288 1048576; do for s in 4 8; do
HYGT_E2E_CHUNK=$ch HYGT_E2E_STREAMS=$s timeout 300 python bench.py --steps 5 --no-cpu --no-extra | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk=$ch streams=$s', round(d['e2e']['value']/1e6,1), 'M vec/s', round(d['e2e']['ms_per_step'],2), 'ms')"
done; done > gpurun_out/exp40.log 2>&1
python - <<'PY' >> gpurun_out/exp40.log 2>&1
import torch, time
x = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
d = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
for name, f in (("H2D", lambda: d.copy_(x, non_blocking=True)), ("D2H", lambda: x.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): f()
    torch.cuda.synchronize()
    print(name, round(5 * (1 << 30) / (time.perf_counter() - t) / 1e9, 1), "GB/s")
PY
cat gpurun_out/exp40.log
