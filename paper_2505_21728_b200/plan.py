"""GPU plans: the batched drop-in for the reference's per-block transform loop.

``HyGTPlan`` replaces the per-class ``HyGTModel`` cache plus the ``hygt::forward`` /
``hygt::inverse`` loop of ``run_apply`` (tools/hygt_main.cpp:143-149); ``FixedPlan`` replaces
``forward_fixed`` / ``inverse_fixed`` (fixedpoint.hpp:191-224, hygt_main.cpp:150-165);
``KLTPlan`` replaces ``klt_forward`` (statistics.hpp:222-224). Device buffers are torch CUDA
tensors (plumbing only); all arithmetic runs in libhygt_gpu.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence, Union

import threading

import numpy as np
import torch

from . import _lib
from .errors import ArgumentError, raise_for
from .model import HyGTModel, ModelBundle, QuantizedHyGTModel, TrigTable

HYGT_PLAN_FORCE_STANDARD = 0x1
HYGT_PLAN_FORCE_FAST = 0x2
HYGT_REUSE_BUCKETS = 0x1


def _check(status: int) -> None:
    if status:
        raise_for(status, _lib.last_error())


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _dev_ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


_CLS_DTYPES = (torch.uint16, torch.int16)


def _ensure(t: Optional[torch.Tensor], name: str, dtypes, numel: Optional[int], device,
            optional: bool = False) -> None:
    """Every tensor handed to the C ABI as a raw pointer is checked here first: a CUDA tensor on
    the plan's device, contiguous, of an accepted dtype and the expected element count.
    Anything else raises ArgumentError before the native call (a mis-sized or host buffer
    would otherwise become an out-of-bounds device write)."""
    if t is None:
        if optional:
            return
        raise ArgumentError(f"{name}: missing tensor")
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ArgumentError(f"{name}: must be a CUDA tensor")
    if device is not None and t.device != torch.device(device):
        raise ArgumentError(f"{name}: must be on {device}, not {t.device}")
    if not t.is_contiguous():
        raise ArgumentError(f"{name}: must be contiguous")
    if dtypes is not None and t.dtype not in dtypes:
        raise ArgumentError(f"{name}: dtype {t.dtype} not in {tuple(dtypes)}")
    if numel is not None and t.numel() != numel:
        raise ArgumentError(f"{name}: {t.numel()} elements, expected {numel}")


def _on_stream(stream):
    """Context that makes `stream` current, so default buffers are allocated (and zero-filled)
    on the stream the kernels run on: the caching allocator then orders their reuse after
    that stream's work."""
    return torch.cuda.stream(stream) if stream is not None else _nullctx()


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _np_ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _models_of(models) -> list:
    if isinstance(models, ModelBundle):
        return [models.dequantized(c) for c in range(models.class_count())]
    if isinstance(models, HyGTModel):
        return [models]
    return list(models)


def _perm_table(models, rounds: int, n: int, inter_round_perms):
    """[C][R][N] gathers + mask: bits 0..R-2 inter-round (BASELINE extension), bit R-1 the
    reference's final sorting permutation (transform.hpp:75-80)."""
    classes = len(models)
    perms = np.tile(np.arange(n, dtype=np.uint16), (classes, rounds, 1))
    mask = 0
    if inter_round_perms is not None:
        ip = np.asarray(inter_round_perms, dtype=np.int64)
        if ip.shape != (classes, rounds - 1, n):
            raise ArgumentError(f"inter_round_perms must have shape {(classes, rounds - 1, n)}")
        perms[:, : rounds - 1, :] = ip
        mask |= (1 << (rounds - 1)) - 1
    if any(m.permutation is not None for m in models):
        for c, m in enumerate(models):
            if m.permutation is not None:
                perms[c, rounds - 1] = m.permutation
        mask |= 1 << (rounds - 1)
    return (np.ascontiguousarray(perms) if mask else None), mask


class _Workspace:
    """Default device workspaces of a plan, one per (host thread, device, stream): calls that share
    a workspace must be stream-ordered, so concurrent callers that pass none never share one."""

    def __init__(self):
        self.bufs = {}
        self.lock = threading.Lock()

    def get(self, nbytes: int, device, stream=None) -> torch.Tensor:
        key = (threading.get_ident(), str(device), _stream_ptr(stream))
        with self.lock:
            buf = self.bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                # allocated and zeroed on the stream the kernels use; a replaced buffer is
                # released through the allocator, which orders its reuse after that stream
                with _on_stream(stream):
                    buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
                self.bufs[key] = buf
            return buf

    def find(self, stream=None) -> Optional[torch.Tensor]:
        """This thread's workspace on `stream` (the current stream by default), if any."""
        sp = _stream_ptr(stream)
        tid = threading.get_ident()
        with self.lock:
            for (t, _, s), buf in self.bufs.items():
                if t == tid and s == sp:
                    return buf
        return None


_KERNEL_NAMES = {
    "stage": "hygt_stage_kernel",
    "jit": "hygt_jit_kernel (NVRTC)",
    "clsjit": "hygt_cls_f (one NVRTC kernel per class; a launch = the chain of per-class grids of one "
              "direction)",
    "cls": "hygt_cls_kernel (a launch = the chain of per-class grids of one direction)",
    "segment": "hygt_segment_kernel",
    "seg2": "hygt_seg2_kernel",
    "tile": "hygt_tile_kernel",
    "bucketed": "hygt_apply_kernel",
    "gemm": "hygt_gemm_kernel / hygt_gemm_ts_kernel at N = 256 (composed per-class operator, tcgen05.mma kind::f16 3-term split)",
}


class HyGTPlan:
    """Batched float HyGT over per-class models.

    models            : HyGTModel, list of HyGTModel (one per class) or ModelBundle
    inter_round_perms : optional [C][R-1][N] gathers applied after rounds 0..R-2
    """

    def __init__(self, models, inter_round_perms=None, flags: int = 0, kernel: str = "auto",
                 allow_nvrtc: bool = True, cta_pairs: bool = True, stage_tile_rows: int = 0):
        """kernel: "auto" (the measured-best family), "butterfly" (rotation kernels only) or
        "tensor" (the composed-operator tensor-core path, N = 64 / 128 / 256); see
        hygt_plan_options in include/hygt_gpu.h for the other options."""
        if kernel not in _lib.KERNELS:
            raise ArgumentError(f"HyGTPlan: kernel must be one of {sorted(_lib.KERNELS)}")
        opts = _lib.plan_options(kernel, allow_nvrtc, cta_pairs, stage_tile_rows)
        models = _models_of(models)
        if not models:
            raise ArgumentError("HyGTPlan: need at least one class")
        log2_n, rounds = models[0].log2_n, models[0].rounds
        for m in models:
            if m.log2_n != log2_n or m.rounds != rounds:
                raise ArgumentError("HyGTPlan: all classes must share log2_n and rounds")
        self.log2_n, self.rounds, self.classes = log2_n, rounds, len(models)
        self.n = 1 << log2_n
        angles = np.ascontiguousarray(np.stack([m.angles for m in models]), dtype=np.float64)
        perms, mask = _perm_table(models, rounds, self.n, inter_round_perms)
        self.perm_mask = mask
        h = C.c_void_p()
        _check(_lib.lib().hygt_plan_create_ex(log2_n, rounds, self.classes, _np_ptr(angles),
                                              _np_ptr(perms), mask, flags, C.byref(opts), C.byref(h)))
        self._h = h
        self._ws = _Workspace()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            try:
                _lib.lib().hygt_plan_destroy(h)
            except Exception:
                pass

    @property
    def handle(self):
        return self._h

    @property
    def input_limit(self) -> float:
        """Largest max|x| per row the plan's fp32 arithmetic keeps finite (hygt_plan_input_limit)."""
        return float(_lib.lib().hygt_plan_input_limit(self._h))

    @property
    def algorithm(self) -> str:
        return "scale-folded" if _lib.lib().hygt_plan_algorithm(self._h) == 1 else "standard"

    @property
    def path(self) -> str:
        """Kernel family serving this plan (include/hygt_gpu.h, hygt_plan_path)."""
        return {0: "bucketed", 1: "tile", 2: "segment", 3: "jit", 4: "stage", 5: "seg2", 6: "cls", 7: "clsjit",
                8: "gemm"}[_lib.lib().hygt_plan_path(self._h)]

    def launches_per_step(self) -> int:
        """Kernels launched by bucket + forward + inverse on this plan (the stage path sorts each
        tile once in hygt_bucket; the tile path sorts inside its kernel; the cls paths launch one
        grid per class and direction after the three bucketing kernels)."""
        path = self.path
        if path in ("cls", "clsjit"):
            return 3 + 2 * self.classes
        return {"tile": 2, "stage": 3}.get(path, 5)  # gemm: 3 bucketing kernels + 2 gemm launches

    def kernel_name(self) -> str:
        """The device kernel(s) one forward or inverse call launches (for reports)."""
        return _KERNEL_NAMES.get(self.path, f"hygt_{self.path}_kernel")

    def workspace_bytes(self, count: int) -> int:
        return _lib.lib().hygt_workspace_bytes(self._h, count)

    def _prep(self, x: torch.Tensor, cls: Optional[torch.Tensor], out: Optional[torch.Tensor],
              stream=None):
        if not isinstance(x, torch.Tensor) or not x.is_cuda:
            raise ArgumentError("HyGTPlan: x must be a CUDA tensor (use apply() for host data)")
        if x.dtype != torch.float32 or x.shape[-1] != self.n or not x.is_contiguous():
            raise ArgumentError("forward: dimension mismatch")
        count = x.numel() // self.n
        _ensure(cls, "HyGTPlan cls", _CLS_DTYPES, count, x.device, optional=True)
        if out is None:
            with _on_stream(stream):
                out = torch.empty_like(x)
        else:
            _ensure(out, "HyGTPlan out", (torch.float32,), x.numel(), x.device)
            if out.shape[-1] != self.n:
                raise ArgumentError("HyGTPlan out: dimension mismatch")
        return count, out

    def _run(self, fn, x, cls, out, stream, workspace, reuse_buckets, energy=None):
        count, out = self._prep(x, cls, out, stream)
        nbytes = self.workspace_bytes(count)
        if workspace is not None:
            _ensure(workspace, "workspace", (torch.uint8,), None, x.device)
            if workspace.numel() < nbytes:
                raise ArgumentError("hygt: workspace too small")
        ws = workspace if workspace is not None else self._ws.get(nbytes, x.device, stream)
        flags = HYGT_REUSE_BUCKETS if reuse_buckets else 0
        args = [self._h, x.data_ptr(), out.data_ptr(), _dev_ptr(cls), count]
        if energy is not None:
            args.append(energy.data_ptr())
        args += [ws.data_ptr(), ws.numel(), flags, _stream_ptr(stream)]
        _check(fn(*args))
        return out

    def forward(self, x, cls=None, out=None, stream=None, workspace=None, reuse_buckets=False):
        """Rows y = forward(x) on the device (asynchronous)."""
        return self._run(_lib.lib().hygt_forward_f32, x, cls, out, stream, workspace, reuse_buckets)

    def inverse(self, y, cls=None, out=None, stream=None, workspace=None, reuse_buckets=False):
        """Rows x = inverse(y) on the device (asynchronous)."""
        return self._run(_lib.lib().hygt_inverse_f32, y, cls, out, stream, workspace, reuse_buckets)

    def forward_energy(self, x, cls, energy, out=None, stream=None, workspace=None,
                       reuse_buckets=False):
        """Forward plus energy[c][i] += sum of y[row][i]^2 over rows of class c (fp64)."""
        _ensure(energy, "forward_energy energy", (torch.float64,), self.classes * self.n, x.device)
        if tuple(energy.shape) != (self.classes, self.n):
            raise ArgumentError("forward_energy: energy must be float64 [classes][N]")
        return self._run(_lib.lib().hygt_forward_energy_f32, x, cls, out, stream, workspace,
                         reuse_buckets, energy=energy)

    def bucket(self, cls, count, workspace, stream=None):
        _ensure(cls, "bucket cls", _CLS_DTYPES, count, None)
        _ensure(workspace, "bucket workspace", (torch.uint8,), None, cls.device)
        if workspace.numel() < self.workspace_bytes(count):
            raise ArgumentError("hygt: workspace too small")
        _check(_lib.lib().hygt_bucket(self._h, _dev_ptr(cls), count, workspace.data_ptr(),
                                      workspace.numel(), _stream_ptr(stream)))

    def sync_status(self, workspace=None, stream=None):
        """Synchronise and raise the device-recorded error (invalid class ids) if any."""
        ws = workspace if workspace is not None else self._ws.find(stream)
        _check(_lib.lib().hygt_sync_status(self._h, _dev_ptr(ws), _stream_ptr(stream)))

    # ---- end-to-end on host buffers (the run_apply call a user makes) ----------------------
    def apply(self, x_host: np.ndarray, cls_host: Optional[np.ndarray] = None,
              inverse: bool = False) -> np.ndarray:
        """Host fp32 rows in, host fp32 rows out (H2D, transform, D2H, status check)."""
        x = torch.from_numpy(np.ascontiguousarray(x_host, dtype=np.float32)).cuda()
        c = None
        if cls_host is not None:
            c = torch.from_numpy(np.ascontiguousarray(cls_host, dtype=np.uint16).view(np.int16)).cuda()
            c = c.view(torch.uint16)
        y = (self.inverse if inverse else self.forward)(x, c)
        self.sync_status()
        return y.cpu().numpy()


class FixedPlan:
    """Bit-exact integer HyGT (forward_fixed / inverse_fixed) over per-class quantized models."""

    def __init__(self, models, table: TrigTable, inter_round_perms=None, allow_nvrtc: bool = True):
        if isinstance(models, ModelBundle):
            models = [models.quantized_model(c) for c in range(models.class_count())]
        elif isinstance(models, QuantizedHyGTModel):
            models = [models]
        models = list(models)
        for m in models:
            if m.angle_bits != table.angle_bits:
                raise ArgumentError("forward_fixed: table/model angle_bits mismatch")
            if m.log2_n != models[0].log2_n or m.rounds != models[0].rounds:
                raise ArgumentError("FixedPlan: all classes must share log2_n and rounds")
        self.log2_n, self.rounds, self.classes = models[0].log2_n, models[0].rounds, len(models)
        self.n = 1 << self.log2_n
        codes = np.ascontiguousarray(np.stack([m.codes for m in models]), dtype=np.uint16)
        perms, mask = _perm_table(models, self.rounds, self.n, inter_round_perms)
        h = C.c_void_p()
        opts = _lib.plan_options(allow_nvrtc=allow_nvrtc)
        _check(_lib.lib().hygt_fixed_plan_create_ex(self.log2_n, self.rounds, self.classes,
                                                    table.angle_bits, table.precision_bits,
                                                    _np_ptr(codes), _np_ptr(perms), mask, C.byref(opts),
                                                    C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            try:
                _lib.lib().hygt_plan_destroy(h)
            except Exception:
                pass

    def _run(self, fn, x, cls, out, stream):
        if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.int64:
            raise ArgumentError("FixedPlan: x must be a CUDA int64 tensor")
        if x.shape[-1] != self.n or not x.is_contiguous():
            raise ArgumentError("fixed transform: dimension mismatch")
        count = x.numel() // self.n
        _ensure(cls, "FixedPlan cls", _CLS_DTYPES, count, x.device, optional=True)
        if out is None:
            with _on_stream(stream):
                out = torch.empty_like(x)
        else:
            _ensure(out, "FixedPlan out", (torch.int64,), x.numel(), x.device)
        bad = C.c_uint64(0)
        st = fn(self._h, x.data_ptr(), out.data_ptr(), _dev_ptr(cls), count, C.byref(bad),
                _stream_ptr(stream))
        self.first_bad = int(bad.value)
        _check(st)
        return out

    @property
    def path(self) -> str:
        return "fixed"

    def launches_per_call(self) -> int:
        """Upper bound of kernels one forward or inverse call launches (bucketing + the
        per-class chain)."""
        return 3 + self.classes

    def forward(self, x, cls=None, out=None, stream=None):
        return self._run(_lib.lib().hygt_forward_i64, x, cls, out, stream)

    def inverse(self, y, cls=None, out=None, stream=None):
        return self._run(_lib.lib().hygt_inverse_i64, y, cls, out, stream)


class KLTPlan:
    """Per-class dense KLT: y = K_c x, x = K_c^T y (statistics.hpp:222-224, matrix.hpp:70-88)."""

    def __init__(self, bases):
        k = np.ascontiguousarray(bases, dtype=np.float64)
        if k.ndim == 2:
            k = k[None]
        self.classes, self.n = k.shape[0], k.shape[1]
        h = C.c_void_p()
        _check(_lib.lib().hygt_klt_plan_create(self.n, self.classes, _np_ptr(k), 0, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            try:
                _lib.lib().hygt_klt_plan_destroy(h)
            except Exception:
                pass

    def workspace_bytes(self, count: int) -> int:
        return _lib.lib().hygt_klt_workspace_bytes(self._h, count)

    def kernel_name(self) -> str:
        if self.n in (64, 128, 256):
            return "hygt_gemm_kernel (per-class grouped GEMM, tcgen05.mma kind::f16 3-term split, CTA pairs)"
        return "klt_tc_kernel (tcgen05.mma kind::tf32, 3xTF32)" if self.n in (16, 32) else "klt_simt_kernel"

    def launches_per_call(self) -> int:
        return 4 if self.classes > 1 else 1  # bucketing (3) + the GEMM kernel (1 with reuse_buckets)

    def _run(self, fn, x, cls, out, stream, workspace=None, reuse_buckets=False):
        if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32:
            raise ArgumentError("KLTPlan: x must be a CUDA float32 tensor")
        if x.shape[-1] != self.n or not x.is_contiguous():
            raise ArgumentError("matrix/vector dimension mismatch")
        count = x.numel() // self.n
        _ensure(cls, "KLTPlan cls", _CLS_DTYPES, count, x.device, optional=True)
        nbytes = max(256, self.workspace_bytes(count))
        if reuse_buckets and workspace is None:
            raise ArgumentError("KLTPlan: reuse_buckets needs the workspace bucket() filled")
        with _on_stream(stream):
            if out is None:
                out = torch.empty_like(x)
            ws = workspace
            if ws is None:
                ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
        _ensure(out, "KLTPlan out", (torch.float32,), x.numel(), x.device)
        _ensure(ws, "KLTPlan workspace", (torch.uint8,), None, x.device)
        if ws.numel() < nbytes:
            raise ArgumentError("hygt_klt: workspace too small")
        _check(fn(self._h, x.data_ptr(), out.data_ptr(), _dev_ptr(cls), count, ws.data_ptr(),
                  ws.numel(), HYGT_REUSE_BUCKETS if reuse_buckets else 0, _stream_ptr(stream)))
        return out

    def bucket(self, cls, count, workspace, stream=None):
        """Group the rows by class once; forward / inverse with reuse_buckets=True then run on
        that grouping (the class dispatch of run_apply is the same for both directions)."""
        _ensure(cls, "KLTPlan cls", _CLS_DTYPES, count, None)
        _ensure(workspace, "KLTPlan workspace", (torch.uint8,), None, cls.device)
        if workspace.numel() < max(256, self.workspace_bytes(count)):
            raise ArgumentError("hygt_klt: workspace too small")
        _check(_lib.lib().hygt_klt_bucket(self._h, _dev_ptr(cls), count, workspace.data_ptr(),
                                          workspace.numel(), _stream_ptr(stream)))

    def forward(self, x, cls=None, out=None, stream=None, workspace=None, reuse_buckets=False):
        """y = K_c x per row on the tensor cores, rows of class c = cls[row]."""
        return self._run(_lib.lib().hygt_klt_forward_f32_ex, x, cls, out, stream, workspace, reuse_buckets)

    def inverse(self, y, cls=None, out=None, stream=None, workspace=None, reuse_buckets=False):
        """x = K_c^T y per row."""
        return self._run(_lib.lib().hygt_klt_inverse_f32_ex, y, cls, out, stream, workspace, reuse_buckets)


# ------------------------------------------------ single-vector drop-ins (transform.hpp) ----
_PLAN_CACHE: dict = {}


def _cached(key, make, owners):
    """Plan cache keyed by object identity; the entry keeps the owning objects alive so an id
    can never be reused by a different model while its plan is cached."""
    hit = _PLAN_CACHE.get(key)
    if hit is not None and all(a is b for a, b in zip(hit[0], owners)):
        return hit[1]
    p = make()
    if len(_PLAN_CACHE) > 64:
        _PLAN_CACHE.clear()
    _PLAN_CACHE[key] = (tuple(owners), p)
    return p


def _model_key(m):
    return (id(m), m.log2_n, m.rounds)


def forward(model: HyGTModel, x) -> np.ndarray:
    """hygt::forward (transform.hpp:72-82) for one vector, computed on the GPU in fp32."""
    v = np.asarray(x, dtype=np.float64).reshape(-1)
    if v.size != model.dimension():
        raise ArgumentError("forward: dimension mismatch")
    plan = _cached(_model_key(model), lambda: HyGTPlan(model), (model,))
    return plan.apply(v[None].astype(np.float32))[0].astype(np.float64)


def inverse(model: HyGTModel, y) -> np.ndarray:
    """hygt::inverse (transform.hpp:86-96) for one vector, computed on the GPU in fp32."""
    v = np.asarray(y, dtype=np.float64).reshape(-1)
    if v.size != model.dimension():
        raise ArgumentError("inverse: dimension mismatch")
    plan = _cached(_model_key(model), lambda: HyGTPlan(model), (model,))
    return plan.apply(v[None].astype(np.float32), inverse=True)[0].astype(np.float64)


def _fixed(model: QuantizedHyGTModel, table: TrigTable, x, inverse_: bool) -> np.ndarray:
    name = "inverse_fixed" if inverse_ else "forward_fixed"
    if table.angle_bits != model.angle_bits:
        raise ArgumentError(f"{name}: table/model angle_bits mismatch")
    v = np.asarray(x, dtype=np.int64).reshape(-1)
    if v.size != model.dimension():
        raise ArgumentError("fixed transform: dimension mismatch")
    plan = _cached((id(model), id(table), "fx"), lambda: FixedPlan(model, table), (model, table))
    t = torch.from_numpy(v[None].copy()).cuda()
    out = plan.inverse(t) if inverse_ else plan.forward(t)
    return out.cpu().numpy()[0]


def forward_fixed(model: QuantizedHyGTModel, table: TrigTable, x) -> np.ndarray:
    """hygt::forward_fixed (fixedpoint.hpp:191-205), bit-exact, on the GPU."""
    return _fixed(model, table, x, False)


def inverse_fixed(model: QuantizedHyGTModel, table: TrigTable, y) -> np.ndarray:
    """hygt::inverse_fixed (fixedpoint.hpp:210-224), bit-exact, on the GPU."""
    return _fixed(model, table, y, True)


# ---- per-class correlation accumulation ------------------------------------------
def correlation(x: torch.Tensor, cls: Optional[torch.Tensor], classes: int,
                sums: Optional[torch.Tensor] = None, counts: Optional[torch.Tensor] = None,
                workspace: Optional[torch.Tensor] = None, stream=None):
    """sums[c] += sum of r r^T over the rows of class c, counts[c] += rows (fp64, on the GPU):
    CorrelationAccumulator::add per class (statistics.hpp:63-99). Returns (sums, counts)."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous():
        raise ArgumentError("correlation: x must be a contiguous CUDA float32 tensor")
    n = x.shape[-1]
    log2_n = n.bit_length() - 1
    if n != 1 << log2_n:
        raise ArgumentError("correlation: row length must be a power of two")
    count = x.numel() // n
    _ensure(cls, "correlation cls", _CLS_DTYPES, count, x.device, optional=True)
    nbytes = _lib.lib().hygt_correlation_workspace_bytes(classes, count)
    with _on_stream(stream):
        if sums is None:
            sums = torch.zeros(classes, n, n, dtype=torch.float64, device=x.device)
        if counts is None:
            counts = torch.zeros(classes, dtype=torch.int64, device=x.device)
        if workspace is None or workspace.numel() < nbytes:
            workspace = torch.zeros(nbytes, dtype=torch.uint8, device=x.device)
    _ensure(sums, "correlation sums", (torch.float64,), classes * n * n, x.device)
    _ensure(counts, "correlation counts", (torch.int64, torch.uint64), classes, x.device)
    _ensure(workspace, "correlation workspace", (torch.uint8,), None, x.device)
    _check(_lib.lib().hygt_correlation_f64(log2_n, classes, x.data_ptr(), _dev_ptr(cls), count,
                                           sums.data_ptr(), counts.data_ptr(), workspace.data_ptr(),
                                           workspace.numel(), _stream_ptr(stream)))
    _check(_lib.lib().hygt_sync_status(None, workspace.data_ptr(), _stream_ptr(stream)))
    return sums, counts


def finalize_correlation(sums: torch.Tensor, counts: torch.Tensor) -> torch.Tensor:
    """phi[c] = sums[c] * (1 / counts[c]) (CorrelationAccumulator::finalize, statistics.hpp:81-94)."""
    inv = 1.0 / counts.to(torch.float64).clamp(min=1)
    return sums * inv[:, None, None]
