import sys, torch, numpy as np, statistics
sys.path.insert(0, '/root/repo')
from paper_2505_21728_b200 import HyGTModel, HyGTPlan
rng = np.random.default_rng(1)
for log2n in (7, 6):
    n = 1 << log2n; R = 4; C = 35
    models = [HyGTModel(log2n, R, rng.uniform(-np.pi, np.pi, R * n * log2n // 2)) for _ in range(C)]
    rows = (1 << 31) // (4 * n)
    x = torch.randn(rows, n, device='cuda') * 16
    cls = torch.randint(0, C, (rows,), device='cuda', dtype=torch.int32).to(torch.int16).view(torch.uint16)
    for kern in ("butterfly", "tensor"):
        plan = HyGTPlan(models, kernel=kern)
        ws = torch.zeros(plan.workspace_bytes(rows), dtype=torch.uint8, device='cuda')
        y = torch.empty_like(x)
        plan.bucket(cls, rows, ws)
        for _ in range(3): plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True); e.record(); ts.append((s, e))
        torch.cuda.synchronize()
        ms = statistics.mean(s.elapsed_time(e) for s, e in ts)
        print(f"N={n} {kern:9s} path={plan.path:8s} {ms:.3f} ms  {rows * (8 * n + 2) / ms / 1e6 / 6546:.3f} of HBM", flush=True)
