mkdir -p gpurun_out
python - <<'PY'
import os, subprocess, numpy as np, sys, time
sys.path.insert(0, ".")
from paper_2505_21728_b200.formats import write_bundle, write_rblk
rng = np.random.default_rng(5)
n, C, R, rows = 16, 35, 3, 1 << 22
cls = rng.integers(0, C, rows).astype(np.uint16); x = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
write_rblk("/tmp/big.rblk", 4, C, cls, x)
A = R * 4 * 8
write_bundle("/tmp/f.hygt", 4, angles=[rng.uniform(-3, 3, A) for _ in range(C)], perms=[rng.permutation(n) for _ in range(C)])
write_bundle("/tmp/q.hygt", 4, codes=[rng.integers(0, 256, A) for _ in range(C)], angle_bits=8, precision_bits=10)
for ar, m in (("float", "/tmp/f.hygt"), ("fixed", "/tmp/q.hygt")):
    for rep in range(2):
        t = time.perf_counter()
        r = subprocess.run(["paper_2505_21728_b200/hygt_gpu_apply", "--model", m, "--data", "/tmp/big.rblk", "--arithmetic", ar, "--out", "/tmp/o.rblk"], capture_output=True, text=True, ) if False else subprocess.run(["paper_2505_21728_b200/hygt_gpu_apply", "--model", m, "--data", "/tmp/big.rblk", "--arithmetic", ar, "--out", "/tmp/o.rblk", "--timing"], capture_output=True, text=True)
        print(ar, rep, round(time.perf_counter() - t, 3), "s", r.stderr.replace("\n", " | "))
PY
