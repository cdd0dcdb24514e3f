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
