"""Device-memory leak probe (development tool): 150 create / run / destroy cycles of float, fixed-point
and KLT plans plus the correlation call; free device memory before and after must match."""
import gc, sys, numpy as np, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2505_21728_b200 import HyGTPlan, HyGTModel, KLTPlan, FixedPlan, QuantizedHyGTModel, TrigTable, correlation
rng = np.random.default_rng(0)
def once(i):
    for log2n, C, R in ((4, 35, 3), (6, 3, 2), (8, 4, 2)):
        n = 1 << log2n
        models = [HyGTModel(log2n, R, rng.uniform(-3, 3, R * log2n * n // 2)) for _ in range(C)]
        p = HyGTPlan(models, allow_nvrtc=False)
        x = torch.randn(3000, n, device="cuda"); c = torch.randint(0, C, (3000,), device="cuda").to(torch.uint16)
        p.inverse(p.forward(x, c), c); p.sync_status()
        del p
    k = np.stack([np.linalg.qr(rng.standard_normal((64, 64)))[0] for _ in range(5)])
    kp = KLTPlan(k); x = torch.randn(3000, 64, device="cuda"); c = torch.randint(0, 5, (3000,), device="cuda").to(torch.uint16)
    kp.forward(x, c); correlation(x, c, 5); del kp
    fp = FixedPlan([QuantizedHyGTModel(4, 2, 8, rng.integers(0, 256, 64)) for _ in range(3)], TrigTable(8, 10), allow_nvrtc=False)
    xi = torch.randint(-1000, 1000, (2000, 16), device="cuda"); ci = torch.randint(0, 3, (2000,), device="cuda").to(torch.uint16)
    fp.forward(xi, ci); del fp
for i in range(5): once(i)
torch.cuda.synchronize(); gc.collect(); torch.cuda.empty_cache()
f0 = torch.cuda.mem_get_info()[0]
for i in range(150): once(i)
torch.cuda.synchronize(); gc.collect(); torch.cuda.empty_cache()
f1 = torch.cuda.mem_get_info()[0]
print(f"free before {f0 / 2**20:.1f} MiB, after 150 create/run/destroy cycles {f1 / 2**20:.1f} MiB, delta {(f0 - f1) / 2**20:.2f} MiB")
