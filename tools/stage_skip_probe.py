"""Staged N = 16 kernel with and without the consumers' arithmetic (debug build, hook
hygt_debug_stage_trace + knob HYGT_STAGE_DEBUG_SKIP): the TMA copy pipeline's own rate (development tool)."""
import ctypes, sys, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2505_21728_b200 import _lib
from paper_2505_21728_b200.synth import make_workload
from paper_2505_21728_b200.plan import HyGTPlan
w = make_workload(2)
rows = w.cfg.count
cls = w.make_classes(rows); x = w.make_rows(rows, cls)
plan = HyGTPlan(w.models, w.perms)
ws = torch.zeros(plan.workspace_bytes(rows), dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
plan.bucket(cls, rows, ws)
lib = _lib.lib()
lib.hygt_debug_stage_trace.argtypes = [ctypes.c_void_p]
tr = torch.zeros(64 * 16, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(label):
    for _ in range(3): plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True)
    ms = 0
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True); b.record(); b.synchronize()
        ms += a.elapsed_time(b)
    print(label, f"{ms / 10 * 1e3:.1f} us", f"{rows * 130 / (ms / 10 * 1e-3) / 1e9:.0f} GB/s")
t("normal")
lib.hygt_debug_stage_trace(ctypes.c_void_p(tr.data_ptr()))
t("debug variant")
_lib.set_knob("HYGT_STAGE_DEBUG_SKIP", 1)
t("debug variant, consumers skip arithmetic (copy pipeline only)")
lib.hygt_debug_stage_trace(None)
