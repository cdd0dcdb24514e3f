"""CPU, world_size 2 over gloo: the multi-GPU host logic of SURVEY.md §8 e1 -- contiguous
shards partition the rows, each rank's per-class energy sums over its shard (computed here by
the oracle in place of the GPU epilogue) all-reduce to the energy of the whole batch, and the
step time reported is the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2505_21728_b200.dist import allreduce_energy, max_over_ranks, shard_range
        rng = np.random.default_rng(3)
        count, classes, log2n, rounds = 1001, 5, 6, 2
        angles = rng.uniform(-np.pi, np.pi, (classes, rounds * 64 * 6 // 2))
        x = (rng.standard_normal((count, 64)) * 16).astype(np.float32)
        cls = rng.integers(0, classes, count).astype(np.uint16)
        a, b = shard_range(count, rank, world)
        e = torch.from_numpy(O.class_energy(log2n, rounds, angles, None, 0, x[a:b], cls[a:b], threads=1))
        allreduce_energy(e)
        t = max_over_ranks(float(rank + 1))
        q.put((rank, (a, b), e.numpy(), t))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_partition():
    from paper_2505_21728_b200.dist import shard_range
    for count in [0, 1, 7, 1000, 1 << 24]:
        for world in [1, 2, 3, 8]:
            spans = [shard_range(count, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            for (a0, b0), (a1, b1) in zip(spans, spans[1:]):
                assert b0 == a1
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_energy_allreduce_world2_gloo():
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(3)
    angles = rng.uniform(-np.pi, np.pi, (5, 2 * 64 * 6 // 2))
    x = (rng.standard_normal((1001, 64)) * 16).astype(np.float32)
    cls = rng.integers(0, 5, 1001).astype(np.uint16)
    full = O.class_energy(6, 2, angles, None, 0, x, cls, threads=1)
    res.sort()
    assert res[0][1] == (0, 501) and res[1][1] == (501, 1001)
    for _, _, e, t in res:
        np.testing.assert_allclose(e, full, rtol=1e-12)
        assert t == 2.0


def _corr_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2505_21728_b200.dist import allreduce_correlation, shard_range
        rng = np.random.default_rng(4)
        x = (rng.standard_normal((777, 16)) * 16).astype(np.float32)
        cls = rng.integers(0, 3, 777).astype(np.uint16)
        a, b = shard_range(777, rank, world)
        s, k = O.correlation(4, 3, x[a:b], cls[a:b])
        s, k = torch.from_numpy(s), torch.from_numpy(k.astype(np.int64))
        allreduce_correlation(s, k)
        q.put((rank, s.numpy(), k.numpy()))
    finally:
        dist.destroy_process_group()


def test_correlation_allreduce_world2_gloo():
    """Per-class second moments of two shards all-reduce to the whole batch's (
    merge_correlation, statistics.hpp:110-120)."""
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_corr_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(4)
    x = (rng.standard_normal((777, 16)) * 16).astype(np.float32)
    cls = rng.integers(0, 3, 777).astype(np.uint16)
    s_full, k_full = O.correlation(4, 3, x, cls)
    for _, s, k in res:
        assert np.abs(s - s_full).max() <= 1e-12 * np.abs(s_full).max()  # fp64 addition order only
        assert np.array_equal(k, k_full.astype(np.int64))


def _helpers_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    from paper_2505_21728_b200 import dist as D
    r, w = D.init_process_group_from_env(torch.device("cpu"))
    try:
        D.barrier()
        a, b = D.shard_range(1001, r, w)
        total = D.sum_over_ranks(b - a)
        t = D.max_over_ranks(0.5 + r)
        q.put((r, w, total, t))
    finally:
        D.destroy()


def test_bench_dist_helpers_world2_gloo():
    """The helpers bench.py's N > 1 path goes through (dist.py): process-group setup from the
    torchrun environment, barrier, the units-processed sum and the max-over-ranks step time."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_helpers_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[:3] for r in res] == [(0, 2, 1001), (1, 2, 1001)]
    assert all(r[3] == 1.5 for r in res)


def _gpu_energy_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_21728_b200 import HyGTPlan
        from paper_2505_21728_b200.dist import shard_range, sharded_forward_energy
        from paper_2505_21728_b200.synth import make_workload
        w = make_workload(5)
        count = 1 << 18
        a, b = shard_range(count, rank, world)
        torch.cuda.set_device(0)
        cls = w.make_classes(b - a, a)
        x = w.make_rows(b - a, cls, a)
        plan = HyGTPlan(w.models)
        e = torch.zeros(35, 256, dtype=torch.float64, device="cuda")
        sharded_forward_energy(plan, x, cls, e)
        plan.sync_status()
        q.put((rank, e.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_energy_two_shards_allreduce_vs_oracle():
    """The GPU forward-with-energy kernel on two shards (two ranks, each a contiguous row range
    generated on the device) plus the all-reduce of dist.sharded_forward_energy equals the
    oracle's energy of the whole batch (config 5 shape, 2^18 rows). The ranks share one GPU
    here (gloo carries the 70 KB exchange; the kernels never wait on each other); on a B200
    node each rank owns a GPU and the same call runs over NCCL."""
    from oracle import oracle as O
    from paper_2505_21728_b200.synth import make_workload
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_energy_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = make_workload(5)
    count = 1 << 18
    cls = w.make_classes(count)
    x = w.make_rows(count, cls)
    ref = O.class_energy(8, 4, w.angles, None, 0, x.cpu().numpy(), cls.cpu().numpy(), hoist=True)
    for _, e in res:
        # the default N = 256 path is the tensor-core one: energies within its stated 2e-6 bar
        # (tests/test_gpu_fullsize.py); the two ranks' tables are identical after the all-reduce
        np.testing.assert_allclose(e, ref, rtol=2e-6)
    assert np.array_equal(res[0][1], res[1][1])
