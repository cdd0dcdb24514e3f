#!/usr/bin/env python3
"""Benchmark of the batched HyGT hot path (BASELINE.json metric: HyGT fwd+inv vectors/s and % of
HBM roofline).

One step = one pass of the hot path over one batch: class bucketing + forward + inverse of every
row of BASELINE config 2 (N=16, C=35 classes, R=3 rounds with inter-round permutations, 2^24
AR(1) rows per GPU; weak scaling over GPUs). Inputs are resident in HBM when the timed region
starts (`value`); `e2e` is the same step through the public host-buffer API with H2D/D2H copies
inside the timed region. `--impl reference` times the reference's own CPU implementation
(oracle/_ref, the unmodified reference headers) on the host cores.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config {1,2,3,4,5}] [--impl ours|reference]

--gpus N without a torchrun environment re-launches this script under torch.distributed.run with
N ranks (one process per GPU, NCCL, 127.0.0.1 rendezvous); under torchrun it reads
RANK/LOCAL_RANK/WORLD_SIZE.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=0, help="override rows per GPU (debug only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config 3 / 5 side measurements")
    ap.add_argument("--verbose", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_traffic(workload: str):
    """DRAM bytes (read + write) of one forward launch of this workload's kernel from the latest
    committed ncu --set full capture (profiles/*/traffic.json), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "traffic.json")), reverse=True):
        try:
            with open(path) as f:
                t = json.load(f).get(workload)
            if t:
                return t["traffic_bytes_per_launch"], os.path.relpath(path, ROOT)
        except Exception:
            pass
    return None, None


def bytes_per_row(n: int, classes: int) -> int:
    """Algorithmic HBM bytes of one direction for one row: N fp32 in + N fp32 out + u16 class id
    (SURVEY.md §8 d2)."""
    return 4 * n + 4 * n + (2 if classes > 1 else 0)


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) is polled from a thread every ~2 ms, so even a region of a few ms gets
    samples; nvidia-smi (-lms 100) is the fallback when NVML is unavailable."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop_flag = threading.Event()
        self.thread = None
        self.proc = None
        self.source = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            return pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        try:
            import pynvml
            h = self._handle()
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop_flag.is_set():
                    try:
                        self.rows.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                          float(mx), int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            self.source = "nvml (2 ms polling)"
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def read():
                for line in self.proc.stdout:
                    parts = [p.strip() for p in line.split(",")]
                    try:
                        self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                    except Exception:
                        pass
            self.thread = threading.Thread(target=read, daemon=True)
            self.thread.start()
            self.source = "nvidia-smi -lms 100"
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.stop_flag.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({nm for r in self.rows for nm, bit in self.REASONS if r[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": self.source}


def dist_setup(gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def respawn(args) -> int:
    """`--gpus N` (N > 1) outside torchrun: re-launch this script with N ranks, one per GPU, over
    torch.distributed.run on 127.0.0.1 (the driver's own launch line), and pass its exit code on."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def config_dict(w, rows, world, scaling):
    """The workload description both arms print (same keys and values, so the driver can check
    that the reference arm ran the same config)."""
    return {"workload": w.cfg.name, "rows_per_gpu": rows, "rows_total": rows * world, "scaling": scaling,
            "N": w.n, "classes": w.cfg.classes, "rounds": w.cfg.rounds,
            "inter_round_perms": w.perms is not None,
            "step": "class bucketing + forward + inverse of every row" if not w.cfg.klt else
                    "class bucketing + KLT forward + KLT inverse of every row",
            "data": "device-generated seeded separable AR(1) rows (synth.py), uniform class ids",
            "parallelism": f"dp{world}"}


# ----------------------------------------------------------------------- CPU reference -----
def host_rows(w, rows, seed=7):
    """Numpy stand-in generator for the CPU arm (same distributions as synth.py: separable AR(1)
    with per-class rho, sigma=16; uniform class ids) so the reference arm touches no GPU code."""
    rng = np.random.default_rng(seed)
    cls = rng.integers(0, w.cfg.classes, rows).astype(np.uint16)
    bs = w.block_size()
    rho = w.rho[cls].astype(np.float64)[:, None]
    q = np.sqrt(1 - rho * rho)
    z = rng.standard_normal((rows, bs, bs))
    for r in range(1, bs):
        z[:, r, :] = rho * z[:, r - 1, :] + q * z[:, r, :]
    for c in range(1, bs):
        z[:, :, c] = rho * z[:, :, c - 1] + q * z[:, :, c]
    return (z.reshape(rows, bs * bs) * w.cfg.sigma).astype(np.float32), cls


def run_reference_sample(w, rows, threads, data=None):
    """Time the reference's hygt::forward + hygt::inverse (oracle/_ref shim over the unmodified
    reference headers) on `rows` rows of the workload with `threads` host threads. Returns s."""
    from oracle import oracle as O
    x, cls = data if data is not None else host_rows(w, rows)
    full, mask = None, 0
    if w.perms is not None:
        full = np.concatenate([w.perms, np.tile(np.arange(w.n, dtype=np.uint16), (w.cfg.classes, 1, 1))], 1)
        mask = (1 << (w.cfg.rounds - 1)) - 1
    t0 = time.perf_counter()
    y = O.ref_apply_batch(w.cfg.log2_n, w.cfg.rounds, w.angles, full, mask, x, cls, False, threads, out="f32")
    O.ref_apply_batch(w.cfg.log2_n, w.cfg.rounds, w.angles, full, mask, y, cls, True, threads, out="f32")
    return time.perf_counter() - t0


def cpu_model() -> str:
    """Host CPU model (SURVEY 8 d4 asks for it next to the core count)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample_rows(n, threads, seconds=1.0):
    """Rows for a bounded CPU sample: the reference does ~3e5 (N=16) / 3e4 (N=64) / 4e3 (N=256)
    fwd+inv rows/s per core, so this is about `seconds` of work on `threads` cores."""
    per_core = {16: 3e5, 64: 3e4, 256: 4e3}.get(n, 1e5)
    return int(min(max(1024, per_core * threads * seconds), (1 << 31) // (4 * n)))


def device_rows(w, rows):
    """The first `rows` rows of the workload exactly as the GPU arm generates them (synth.py's
    counter-based device generator, row0 = 0), copied to host memory; None without a GPU."""
    try:
        import torch
        if not torch.cuda.is_available():
            return None
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        cls = w.make_classes(rows)
        x = w.make_rows(rows, cls)
        out = (x.cpu().numpy(), cls.cpu().numpy())
        del x, cls
        torch.cuda.empty_cache()
        return out
    except Exception:
        return None


def impl_reference(args):
    """The reference arm: the reference's own CPU implementation (hygt::forward + hygt::inverse
    per row, unmodified headers compiled into oracle/_ref) on all host threads, on the same
    workload rows the GPU arm transforms. Each step is the whole batch when that takes a few
    seconds (configs 1 and 2), else a bounded prefix of it (stated in cpu_baseline.sample)."""
    rank, world, local = dist_setup(args.gpus)
    if rank != 0:
        return 0
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(args.config)
    threads = os.cpu_count() or 1
    full = args.rows or w.cfg.count
    rows = min(full, cpu_sample_rows(w.n, threads, seconds=6.0))
    data = device_rows(w, rows)
    source = "the GPU arm's device-generated rows [0, rows)"
    if data is None:
        data = host_rows(w, rows)
        source = "host-generated rows of the same distributions (no GPU to generate them)"
    times = []
    for i in range(args.warmup + args.steps):
        t = run_reference_sample(w, rows, threads, data)
        if i >= args.warmup:
            times.append(t)
    t = statistics.median(times)
    v = rows / t
    cfg = config_dict(w, full, world, "weak")
    line = {
        "impl": "reference", "metric": "HyGT fwd+inv vectors/s", "value": v, "unit": "vectors/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": v, "unit": "vectors/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{rows} of the {full} rows per step ({'the whole batch' if rows == full else 'a prefix'}; "
                                   f"{source}), hygt::forward+hygt::inverse per row (unmodified reference "
                                   f"headers, g++ -O2), {threads} std::threads; rank 0 only"},
        "e2e": {"value": v, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- ours --------
def timed_region(steps, stream, local, step_fn, world, dev):
    """K device-timed steps (CUDA events on the launching stream, a 256 MiB L2 flush before
    each, barrier + synchronize on both sides), clocks sampled during the region. Returns
    (mean ms per step over ranks' max, per-step event lists, clocks summary)."""
    import torch
    from paper_2505_21728_b200 import dist as D
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = []
    total_ms = 0.0
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        D.barrier()
        for _ in range(steps):
            l2_flush.zero_()  # inputs are > L2 already; flush anyway so no step starts L2-warm
            start.record(stream)
            evs.append(step_fn())
            stop.record(stream)
            stop.synchronize()
            total_ms += start.elapsed_time(stop)
        torch.cuda.synchronize()
        D.barrier()
    ms = D.max_over_ranks(total_ms / steps, device=dev)
    return ms, evs, clocks.summary()


def measure_klt(args, rank, world, local, dev, steps, warmup):
    """Config 4: the dense per-class KLT comparison path on config 3's rows (grouped per-class
    GEMM on the tensor cores); vectors/s, GB/s, TFLOP/s and the KLT/HyGT footprint ratio."""
    import torch
    from paper_2505_21728_b200 import KLTPlan, TransformKind, memory_footprint
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(4)
    rows = args.rows or w.cfg.count
    cls = w.make_classes(rows, rank * rows)
    x = w.make_rows(rows, cls, rank * rows)
    y = torch.empty_like(x)
    xr = torch.empty_like(x)
    plan = KLTPlan(w.klt_bases())
    ws = torch.zeros(max(256, plan.workspace_bytes(rows)), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    def step():  # as the HyGT step: class bucketing once, then both directions on that grouping
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        plan.bucket(cls, rows, ws)
        ev[1].record(stream)
        plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True)
        ev[2].record(stream)
        plan.inverse(y, cls, out=xr, workspace=ws, reuse_buckets=True)
        ev[3].record(stream)
        return ev
    for _ in range(max(warmup, 3)):
        step()
    torch.cuda.synchronize()
    ms, evs, clocks = timed_region(steps, stream, local, step, world, dev)
    bk = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    fw = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    inv = statistics.mean(e[2].elapsed_time(e[3]) for e in evs)
    n = w.n
    hbm, hbm_kind = peaks()
    bpr = bytes_per_row(n, w.cfg.classes)
    launch_ms = (fw + inv) / 2
    achieved = rows * bpr / (launch_ms * 1e-3) / 1e9
    flops = 2.0 * n * n  # algorithmic per row and direction
    err = (xr - x).abs().max().item() / x.abs().max().item()
    traffic, traffic_src = measured_traffic(w.cfg.name) if rows == w.cfg.count else (None, None)
    return {
        "workload": w.cfg.name, "metric": "KLT fwd+inv vectors/s (config 4 comparison path)",
        "value": rows * world / (ms * 1e-3), "unit": "vectors/s", "ms_per_step": ms, "steps": steps,
        "warmup": max(warmup, 3), "rows_per_gpu": rows, "scaling": "weak", "N": n, "classes": w.cfg.classes,
        "kernel": plan.kernel_name(),
        "breakdown_ms": {"bucket": bk, "forward": fw, "inverse": inv},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({hbm_kind})"},
        "tflops_algorithmic": rows * flops / (launch_ms * 1e-3) / 1e12,
        "memory_ratio_units": memory_footprint(TransformKind.klt, 6, 1, 35) /
                              memory_footprint(TransformKind.hygt, 6, 4, 35),
        "memory_ratio_fp32_bytes_vs_fp32_cs_tables": (35 * 64 * 64 * 4) / (35 * 768 * 8),
        "roundtrip_max_rel": err, "clocks": clocks, "gpu_launches": (3 + 2) * steps,
    }


def measure_fixed(args, rank, world, local, dev, steps, warmup, config=2):
    """The bit-exact fixed-point path (forward_fixed / inverse_fixed, 8-bit codes, TrigTable(8,
    10)) on a config's shape with int64 rows (|x| <= 2^20, rounded from the AR(1) rows)."""
    import torch
    from paper_2505_21728_b200 import FixedPlan, TrigTable, quantize_model
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(config)
    rows = args.rows or w.cfg.count
    table = TrigTable(8, 10)
    plan = FixedPlan([quantize_model(m, 8) for m in w.models], table, w.perms)
    cls = w.make_classes(rows, rank * rows)
    x = torch.round(w.make_rows(rows, cls, rank * rows)).to(torch.int64).clamp_(-(1 << 20), 1 << 20)
    y = torch.empty_like(x)
    xr = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    for _ in range(max(warmup, 3)):
        plan.forward(x, cls, out=y)
        plan.inverse(y, cls, out=xr)
    torch.cuda.synchronize()

    def step():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        plan.forward(x, cls, out=y)
        ev[1].record(stream)
        plan.inverse(y, cls, out=xr)
        ev[2].record(stream)
        return ev
    ms, evs, clocks = timed_region(steps, stream, local, step, world, dev)
    fw = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    inv = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    n = w.n
    hbm, hbm_kind = peaks()
    bpr = 8 * n * 2 + (2 if w.cfg.classes > 1 else 0)
    launch_ms = (fw + inv) / 2
    achieved = rows * bpr / (launch_ms * 1e-3) / 1e9
    return {
        "workload": w.cfg.name + "_fixed_b8_p10", "metric": "fixed-point HyGT fwd+inv vectors/s (bit-exact)",
        "value": rows * world / (ms * 1e-3), "unit": "vectors/s", "ms_per_step": ms, "steps": steps,
        "warmup": max(warmup, 3), "rows_per_gpu": rows, "scaling": "weak", "N": n, "classes": w.cfg.classes,
        "dtype": "int64 rows, int32/int64 arithmetic", "kernel_path": plan.path,
        "breakdown_ms": {"forward (incl. bucketing, status read-back)": fw, "inverse": inv},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": None, "note": "bound by the integer multiply pipe, not HBM (DESIGN.md 5.8)"},
        "roundtrip_exact_rows_frac": float((xr == x).all(1).double().mean().item()),
        "clocks": clocks, "gpu_launches": plan.launches_per_call() * 2 * steps,
    }


def measure_device(config, args, rank, world, local, dev, steps, warmup, strong=False):
    """Device-timed bucket + forward + inverse steps of one config (inputs resident in HBM, a
    256 MiB L2 flush before each step, CUDA events on the launching stream, max over ranks).
    Weak scaling: every rank transforms the config's full row count; strong: the config's rows
    are sharded across the ranks (dist.shard_range). Config 5 also all-reduces the per-class
    energies (the one exchange step, dist.allreduce_energy). Returns (summary, state)."""
    import torch
    from paper_2505_21728_b200 import HyGTPlan
    from paper_2505_21728_b200 import dist as D
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(config)
    total = args.rows or w.cfg.count
    if strong:
        row0, row1 = D.shard_range(total, rank, world)
    else:
        row0, row1 = rank * total, (rank + 1) * total
    rows = row1 - row0
    n = w.n
    cls = w.make_classes(rows, row0)
    x = w.make_rows(rows, cls, row0)
    y = torch.empty_like(x)
    xr = torch.empty_like(x)
    plan = HyGTPlan(w.models, w.perms)
    ws = torch.zeros(plan.workspace_bytes(rows), dtype=torch.uint8, device=dev)
    energy = torch.zeros(w.cfg.classes, n, dtype=torch.float64, device=dev) if w.cfg.energy else None
    stream = torch.cuda.current_stream()

    def step(timed=True):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if timed else None
        rec = (lambda k: ev[k].record(stream)) if timed else (lambda k: None)
        rec(0)
        plan.bucket(cls, rows, ws)
        rec(1)
        if energy is not None:
            energy.zero_()
            plan.forward_energy(x, cls, energy, out=y, workspace=ws, reuse_buckets=True)
        else:
            plan.forward(x, cls, out=y, workspace=ws, reuse_buckets=True)
        rec(2)
        plan.inverse(y, cls, out=xr, workspace=ws, reuse_buckets=True)
        rec(3)
        if energy is not None:
            D.allreduce_energy(energy)  # 35 x 256 fp64 over NCCL at N > 1 (a no-op at N = 1)
        rec(4)
        return ev

    for _ in range(max(warmup, 3)):
        step(False)
    plan.sync_status(ws)
    torch.cuda.synchronize()
    D.barrier()
    ms, evs, clocks = timed_region(steps, stream, local, step, world, dev)
    t_bucket = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    t_fwd = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    t_inv = statistics.mean(e[2].elapsed_time(e[3]) for e in evs)
    t_ar = statistics.mean(e[3].elapsed_time(e[4]) for e in evs)
    plan.sync_status(ws)
    total_rows = D.sum_over_ranks(rows, device=dev)

    hbm, hbm_kind = peaks()
    bpr = bytes_per_row(n, w.cfg.classes)
    launch_ms = (t_fwd + t_inv) / 2  # the fwd and inv apply kernels (same kernel family)
    achieved = rows * bpr / (launch_ms * 1e-3) / 1e9
    traffic, traffic_src = measured_traffic(w.cfg.name) if rows == w.cfg.count else (None, None)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": plan.kernel_name() + " (mean of the forward and inverse launches)",
                "bytes_per_launch": rows * bpr, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({hbm_kind})"}
    out = {"workload": w.cfg.name, "value": total_rows / (ms * 1e-3), "unit": "vectors/s",
           "ms_per_step": ms, "steps": steps, "warmup": max(warmup, 3), "rows_per_gpu": rows,
           "scaling": "strong" if strong else "weak", "N": n, "classes": w.cfg.classes,
           "rounds": w.cfg.rounds, "inter_round_perms": w.perms is not None,
           "energy_allreduce": bool(w.cfg.energy), "algorithm": plan.algorithm, "kernel_path": plan.path,
           "breakdown_ms": {"bucket": t_bucket, "forward": t_fwd, "inverse": t_inv,
                            **({"energy_allreduce": t_ar} if energy is not None else {})},
           "roofline": roofline, "clocks": clocks,
           "gpu_launches": plan.launches_per_step() * steps}
    return out, (w, plan, x, cls, rows, stream)


def impl_ours(args):
    import torch
    from paper_2505_21728_b200 import dist as D
    rank, world, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    D.init_process_group_from_env(dev)
    if args.config == 4:
        res = measure_klt(args, rank, world, local, dev, args.steps, args.warmup)
        if rank == 0:
            line = {k: res[k] for k in ("metric", "value", "unit", "ms_per_step", "roofline", "clocks", "gpu_launches")}
            line.update({"n_gpus": world, "steps": args.steps, "warmup": res["warmup"], "higher_is_better": True,
                         "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                         "config": {"workload": res["workload"], "rows_per_gpu": res["rows_per_gpu"],
                                    "N": res["N"], "classes": res["classes"], "kernel": res["kernel"]},
                         "tflops_algorithmic": res["tflops_algorithmic"],
                         "memory_ratio_units": res["memory_ratio_units"]})
            print(json.dumps(line), flush=True)
        D.destroy()
        return 0
    res, (w, plan, x, cls, rows, stream) = measure_device(args.config, args, rank, world, local, dev,
                                                          args.steps, args.warmup)
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(plan, w, x, cls, rows, dev, stream, args, world)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        srows = min(rows, cpu_sample_rows(w.n, threads, seconds=5.0))  # never more rows than the batch holds
        t = run_reference_sample(w, srows, threads, (x[:srows].cpu().numpy(), cls[:srows].cpu().numpy()))
        cpu = {"value": srows / t, "unit": "vectors/s", "cores": threads, "kind": "reference",
               "cpu_model": cpu_model(),
               "sample": f"the first {srows} rows of the timed batch ({w.cfg.name}): hygt::forward+hygt::inverse "
                         f"per row (unmodified reference headers via oracle/_ref, g++ -O2), {threads} threads"}
    del plan, x, cls
    # The metric names N = 16 / 64 / 256: the default run also times configs 1, 3 and 5 (config 5
    # weak and, at N > 1, strong), the config-4 KLT comparison and the fixed-point path, each
    # under the same rules with its own clocks, beside the headline.
    others = []
    if args.config == 2 and not args.no_extra and not args.rows:
        k = max(3, min(args.steps, 10))
        # config 5 (tensor-core heavy, runs into the board's power cap) goes last, and every
        # measurement starts after a short idle so no run inherits the previous one's clocks
        jobs = [("hygt", 1, False), ("hygt", 3, False), ("klt", 4, False), ("fixed", 2, False), ("hygt", 5, False)]
        if world > 1:
            jobs.append(("hygt", 5, True))
        for kind, c, strong in jobs:
            torch.cuda.empty_cache()
            time.sleep(3.0)
            if kind == "hygt":
                o, _ = measure_device(c, args, rank, world, local, dev, k, args.warmup, strong=strong)
            elif kind == "klt":
                o = measure_klt(args, rank, world, local, dev, k, args.warmup)
            else:
                o = measure_fixed(args, rank, world, local, dev, k, args.warmup, config=c)
            others.append(o)
            torch.cuda.empty_cache()
    if rank == 0:
        cfg = config_dict(w, rows, world, res["scaling"])
        cfg.update({"l2": "inputs larger than L2 (>=1 GiB per array) and a 256 MiB L2 flush between steps",
                    "algorithm": res["algorithm"], "kernel_path": res["kernel_path"]})
        line = {
            "metric": "HyGT fwd+inv vectors/s", "value": res["value"], "unit": "vectors/s",
            "n_gpus": world, "steps": args.steps, "warmup": res["warmup"],
            "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": res["scaling"],
            "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (device-generated separable AR(1) rows, seeded)",
            "config": cfg,
            "breakdown_ms": res["breakdown_ms"],
            "roofline": res["roofline"],
            "clocks": res["clocks"],
            "gpu_launches": res["gpu_launches"],
        }
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        if others:
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    D.destroy()
    return 0


def measure_e2e(plan, w, x, cls, rows, dev, stream, args, world=1):
    """Same step through the host-buffer API: pinned host x/cls -> device -> bucket + fwd + inv ->
    host y and reconstruction, chunked over two streams so copies overlap compute."""
    import torch
    from paper_2505_21728_b200.pipeline import HostPipeline
    xh = x.cpu().pin_memory()
    ch = cls.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    rh = torch.empty_like(xh).pin_memory()
    pipe = HostPipeline(plan, rows_per_chunk=min(rows, int(os.environ.get("HYGT_E2E_CHUNK", 1 << 20))), device=dev,
                        streams=int(os.environ.get("HYGT_E2E_STREAMS", 4)))
    for _ in range(2):
        pipe.roundtrip(xh, ch, yh, rh)
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 5))
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        pipe.roundtrip(xh, ch, yh, rh)
    stop.record(stream)
    stop.synchronize()
    t = start.elapsed_time(stop) * 1e-3 / steps
    from paper_2505_21728_b200 import dist as D
    t = D.max_over_ranks(t, device=dev)
    n = w.n
    h2d = rows * n * 4 + rows * 2
    d2h = 2 * rows * n * 4
    return {"value": rows * world / t, "unit": "vectors/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": t * 1e3,
            "path": "HostPipeline.roundtrip (pinned host in -> H2D -> bucket+fwd+inv -> D2H coefficients and reconstruction)"}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return respawn(args)
    if args.impl == "reference":
        return impl_reference(args)
    return impl_ours(args)


if __name__ == "__main__":
    sys.exit(main())
