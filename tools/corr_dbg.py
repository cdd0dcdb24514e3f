import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2505_21728_b200._lib as L
from paper_2505_21728_b200 import correlation
from oracle import oracle as O
rng = np.random.default_rng(68)
for n_log, count in [(8, 3000), (7, 3000)]:
    n = 1 << n_log
    x = (rng.standard_normal((count, n)) * 16).astype(np.float32)
    cls = rng.integers(0, 2, count).astype(np.uint16)
    ref_s, ref_k = O.correlation(n_log, 2, x, cls)
    for dbg in [0, 0, 0]:
        L.set_knob("HYGT_CORR_DBG", dbg)
        s, k = correlation(torch.from_numpy(x).cuda(), torch.from_numpy(cls).cuda(), 2)
        s = s.cpu().numpy()
        err = np.abs(s - ref_s)
        bad = np.argwhere(err > 1e-9 * np.abs(ref_s).max())
        blocks = sorted(set((int(a) // 64, int(b) // 64) for _, a, b in bad))
        print(n, "dbg", dbg, "maxerr", err.max() / np.abs(ref_s).max(), "bad blocks", blocks[:20])
