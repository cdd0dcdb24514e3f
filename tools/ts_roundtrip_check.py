import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2505_21728_b200._lib as L
from paper_2505_21728_b200 import HyGTModel, HyGTPlan
for dbg in [0, 8, 0, 8]:
    L.clear_knobs()
    if dbg: L.set_knob("HYGT_GEMM_DBG", dbg)
    rng = np.random.default_rng(7)
    classes = 400
    models = [HyGTModel(8, 2, rng.uniform(-np.pi, np.pi, 2 * 8 * 128)) for _ in range(classes)]
    plan = HyGTPlan(models, kernel="tensor")
    x = torch.from_numpy((rng.standard_normal((20000, 256)) * 16).astype(np.float32)).cuda()
    cls = torch.from_numpy(rng.integers(0, classes, 20000).astype(np.uint16)).cuda()
    y = plan.forward(x, cls)
    z = plan.inverse(y, cls)
    e = torch.zeros(classes, 256, dtype=torch.float64, device="cuda")
    y2 = plan.forward_energy(x, cls, e)
    z2 = plan.inverse(y2, cls)
    torch.cuda.synchronize()
    print(f"dbg {dbg}: round trip max err {float((z - x).abs().max()):.3e}, with energy {float((z2 - x).abs().max()):.3e}, fwd vs fwd+energy {float((y - y2).abs().max()):.3e}", flush=True)
