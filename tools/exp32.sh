# clsjit: PTX bodies vs C++ bodies (plan creation time and speed)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "seg2_path or golden_float or config_shapes" > gpurun_out/pt_ptx.log 2>&1; echo rc=$? >> gpurun_out/pt_ptx.log
tail -2 gpurun_out/pt_ptx.log
for m in 1 0; do
HYGT_CLS_PTX=$m python - <<'PY'
import time, os
import numpy as np
from paper_2505_21728_b200 import HyGTModel, HyGTPlan
rng = np.random.default_rng(5)
t = time.time()
plan = HyGTPlan([HyGTModel(6, 4, rng.uniform(-3, 3, 4 * 6 * 32)) for _ in range(35)],
                np.stack([np.stack([rng.permutation(64) for _ in range(3)]) for _ in range(35)]))
print("ptx", os.environ["HYGT_CLS_PTX"], "plan creation", round(time.time() - t, 2), "s", plan.path, os.cpu_count(), "cpus")
PY
HYGT_CLS_PTX=$m python tools/kbench.py 6:4:35:perm 5:3:35:perm
done
