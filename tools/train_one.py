"""One trainer launch (the N=64 R=3 acceptance case, restarts 4) for ncu."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2505_21728_b200 import train as T
a = 0.95 ** np.abs(np.subtract.outer(np.arange(8), np.arange(8)))
m, r = T.optimize(np.kron(a, a), 6, 3, T.OptimizerConfig(restarts=4, seed=1, max_sweeps=int(sys.argv[1]) if len(sys.argv) > 1 else 50))
print(r.restart_gains_db)
