"""ctypes binding of libhygt_gpu.so (include/hygt_gpu.h).

The product path has no CPU fallback: if the CUDA library is missing or fails to load, every
entry point raises. Build it with ``python -c "import __graft_entry__ as g; g.build()"``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhygt_gpu.so")

_p = C.c_void_p
_i = C.c_int
_u32 = C.c_uint32
_u64 = C.c_uint64
_sz = C.c_size_t
_f = C.c_float

# Every symbol include/hygt_gpu.h declares, with its ctypes signature (restype, argtypes).
SIGNATURES = {
    "hygt_last_error": (_i, [C.c_char_p, _sz]),
    "hygt_plan_create": (_i, [_i, _i, _i, _p, _p, _u32, _u32, C.POINTER(_p)]),
    "hygt_plan_create_ex": (_i, [_i, _i, _i, _p, _p, _u32, _u32, _p, C.POINTER(_p)]),
    "hygt_plan_destroy": (_i, [_p]),
    "hygt_plan_algorithm": (_i, [_p]),
    "hygt_plan_input_limit": (C.c_double, [_p]),
    "hygt_plan_path": (_i, [_p]),
    "hygt_workspace_bytes": (_sz, [_p, _u64]),
    "hygt_bucket": (_i, [_p, _p, _u64, _p, _sz, _p]),
    "hygt_forward_f32": (_i, [_p, _p, _p, _p, _u64, _p, _sz, _u32, _p]),
    "hygt_inverse_f32": (_i, [_p, _p, _p, _p, _u64, _p, _sz, _u32, _p]),
    "hygt_forward_energy_f32": (_i, [_p, _p, _p, _p, _u64, _p, _p, _sz, _u32, _p]),
    "hygt_sync_status": (_i, [_p, _p, _p]),
    "hygt_fixed_plan_create": (_i, [_i, _i, _i, _i, _i, _p, _p, _u32, C.POINTER(_p)]),
    "hygt_fixed_plan_create_ex": (_i, [_i, _i, _i, _i, _i, _p, _p, _u32, _p, C.POINTER(_p)]),
    "hygt_forward_i64": (_i, [_p, _p, _p, _p, _u64, C.POINTER(_u64), _p]),
    "hygt_inverse_i64": (_i, [_p, _p, _p, _p, _u64, C.POINTER(_u64), _p]),
    "hygt_correlation_workspace_bytes": (_sz, [_i, _u64]),
    "hygt_correlation_f64": (_i, [_i, _i, _p, _p, _u64, _p, _p, _p, _sz, _p]),
    "hygt_optimize_f64": (_i, [_i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "hygt_klt_plan_create": (_i, [_i, _i, _p, _u32, C.POINTER(_p)]),
    "hygt_klt_plan_destroy": (_i, [_p]),
    "hygt_klt_workspace_bytes": (_sz, [_p, _u64]),
    "hygt_klt_forward_f32": (_i, [_p, _p, _p, _p, _u64, _p, _sz, _p]),
    "hygt_klt_inverse_f32": (_i, [_p, _p, _p, _p, _u64, _p, _sz, _p]),
    "hygt_klt_bucket": (_i, [_p, _p, _u64, _p, _sz, _p]),
    "hygt_klt_forward_f32_ex": (_i, [_p, _p, _p, _p, _u64, _p, _sz, _u32, _p]),
    "hygt_klt_inverse_f32_ex": (_i, [_p, _p, _p, _p, _u64, _p, _sz, _u32, _p]),
    "hygt_synth_rows_f32": (_i, [_p, _u64, _u64, _i, _p, _p, _i, _f, _f, _f, _f, _u64, _p]),
    "hygt_synth_classes": (_i, [_p, _u64, _u64, _i, _u64, _p]),
}

_LIB = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load (once) and return the CUDA library; raises if it is not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def last_error() -> str:
    buf = C.create_string_buffer(512)
    lib().hygt_last_error(buf, 512)
    return buf.value.decode(errors="replace")


class PlanOptions(C.Structure):
    """hygt_plan_options (include/hygt_gpu.h)."""
    _fields_ = [("size", C.c_uint32), ("kernel", C.c_int), ("allow_nvrtc", C.c_int),
                ("cta_pairs", C.c_int), ("stage_tile_rows", C.c_int)]


KERNELS = {"auto": 0, "butterfly": 1, "tensor": 2}


def plan_options(kernel="auto", allow_nvrtc=True, cta_pairs=True, stage_tile_rows=0):
    o = PlanOptions()
    o.size = C.sizeof(PlanOptions)
    o.kernel = KERNELS[kernel]
    o.allow_nvrtc = 1 if allow_nvrtc else 0
    o.cta_pairs = 1 if cta_pairs else 0
    o.stage_tile_rows = int(stage_tile_rows)
    return o


# ---- test hook (not part of the public header): development knobs of the kernel selection ----
def set_knob(name: str, value) -> None:
    """Sets a development knob (hygt_knobs.h) for plans created afterwards in this process."""
    fn = lib().hygt_debug_set_knob
    fn.argtypes = [C.c_char_p, C.c_int]
    fn.restype = None
    fn(name.encode(), int(value))


def clear_knobs() -> None:
    fn = lib().hygt_debug_clear_knobs
    fn.argtypes = []
    fn.restype = None
    fn()
