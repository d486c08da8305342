"""Multi-GPU front-end host logic (paper_0811_3448_b200.dist) on CPU.

The splitter choice, tie division, split sizes and the all-to-all-v plumbing
run for real over gloo with world_size 2 and 3; the per-rank device steps
(sampling, destination partition, local sort) are stood in by a numpy
LocalOps defined here (test infrastructure), so no GPU is needed.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0811_3448_b200.dist import boundaries, choose_splitters, dist_sort, send_counts


def test_boundaries_cut_only_tie_classes():
    # 2 ranks, 3 classes: [below s0, == s0, above s0]
    cc = np.array([[4, 10, 2], [0, 10, 0]])  # rank 0 / rank 1 class counts
    B = boundaries(cc, 2)
    assert B[0] == 0 and B[2] == 26 and B[1] == 13  # lands inside the tie class
    assert send_counts(cc, B, 0) == [13, 3] and send_counts(cc, B, 1) == [0, 10]
    cc = np.array([[10, 0, 3], [7, 0, 6]])  # boundary lands in an even class
    B = boundaries(cc, 2)
    assert B[1] in (0, 17)


def test_boundaries_many_ranks_balanced_uniform():
    rng = np.random.default_rng(0)
    R = 8
    cc = rng.integers(1000, 1100, size=(R, 2 * R - 1))
    cc[:, 1::2] = rng.integers(0, 3, size=(R, R - 1))  # few exact ties
    B = boundaries(cc, R)
    assert np.all(np.diff(B) >= 0) and B[-1] == cc.sum()
    for r in range(R):
        sc = send_counts(cc, B, r)
        assert sum(sc) == cc[r].sum()
    recv = [sum(send_counts(cc, B, s)[d] for s in range(R)) for d in range(R)]
    assert recv == np.diff(B).tolist()


def test_choose_splitters():
    s = np.arange(100, dtype=np.uint32)
    assert choose_splitters(s, 4).tolist() == [25, 50, 75]
    assert choose_splitters(s, 1).size == 0


class NumpyOps:
    """CPU stand-in for CudaOps (unsigned full-width keys): test infrastructure."""

    def __init__(self, width):
        self.width = width

    def sample(self, keys, count):
        n = keys.numel()
        if n == 0 or count == 0:
            return keys[:0].clone()
        idx = [((2 * i + 1) * n) // (2 * count) for i in range(count)]
        return keys[idx].clone()

    def sort_samples(self, samples):
        u = _u(samples)
        return _t(np.sort(u), samples.dtype)

    def split(self, keys, values, splitters, nranks):
        k = _u(keys)
        sp = _u(splitters)
        lt = (sp[None, :] < k[:, None]).sum(axis=1)
        eq = (sp[None, :] == k[:, None]).any(axis=1)
        cls = 2 * lt + eq
        order = np.argsort(cls, kind="stable")
        counts = np.bincount(cls, minlength=2 * nranks - 1)
        out_v = values[torch.from_numpy(order)] if values is not None else None
        return _t(k[order], keys.dtype), out_v, torch.from_numpy(counts.astype(np.int64))

    def sort(self, keys, values):
        k = _u(keys)
        order = np.argsort(k, kind="stable")
        return _t(k[order], keys.dtype), (values[torch.from_numpy(order)] if values is not None else None)


def _u(t):
    a = t.numpy()
    return a.view(np.uint32 if a.itemsize == 4 else np.uint64)


def _t(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32 if a.itemsize == 4 else np.int64)).to(dtype)


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(100 + rank)
        n = 5000 + 137 * rank
        if kind == "uniform":
            k = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
        elif kind == "heavy":  # one value holds ~half the keys (Zipf-like tie)
            k = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
            k[rng.random(n) < 0.5] = 12345
        else:  # sorted shards: rank r holds a high range
            k = np.sort(rng.integers(0, 2 ** 20, n, dtype=np.uint64).astype(np.uint32)) + np.uint32(rank << 20)
        vals = torch.arange(n, dtype=torch.int64) + (rank << 32)
        res = dist_sort(_t(k, torch.int32), vals, width=32, ops=NumpyOps(32))
        q.put((rank, _u(res.keys).copy(), res.values.numpy().copy(), k))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,kind", [(2, "uniform"), (2, "heavy"), (3, "sorted"), (3, "heavy")])
def test_dist_sort_gloo(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda t: t[0])
    keys_all = np.concatenate([g[1] for g in got])
    vals_all = np.concatenate([g[2] for g in got])
    inputs = np.concatenate([g[3] for g in got])
    # global order: concatenation over ranks is the sorted whole
    assert np.array_equal(keys_all, np.sort(inputs))
    # pairs preserved and stable across ranks: (key, source rank, index) order
    src_rank = vals_all >> 32
    src_idx = vals_all & 0xFFFFFFFF
    offs = np.cumsum([0] + [g[3].size for g in got])
    assert np.array_equal(inputs[offs[src_rank] + src_idx], keys_all)
    order = np.argsort(inputs, kind="stable")
    assert np.array_equal(offs[src_rank] + src_idx, order)
    # balance: every rank within one tie class of an even share
    sizes = [g[1].size for g in got]
    if kind == "uniform":
        assert max(sizes) - min(sizes) <= 0.05 * inputs.size


@pytest.mark.parametrize("R,kind", [(2, "uniform"), (3, "heavy"), (4, "sorted"), (8, "heavy")])
def test_exchange_plan_matches_all_to_all(R, kind):
    """The fused exchange's placement rule (gpos = shard class-major position +
    delta[class], destination by bounds) yields exactly the receive buffers of
    partition + all-to-all-v (source-rank order within each destination, up to
    the class-major interleave that the stable local sort absorbs) -- checked
    here on the full element identity, with numpy shards for every rank."""
    from paper_0811_3448_b200.dist import exchange_plan

    rng = np.random.default_rng(R * 7 + len(kind))
    shards = []
    for r in range(R):
        n = 3000 + 211 * r
        k = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
        if kind == "heavy":
            k[rng.random(n) < 0.6] = 777
        elif kind == "sorted":
            k = np.sort(k >> np.uint32(4)) + np.uint32(r << 28)
        shards.append(k)
    allk = np.concatenate(shards)
    spl = choose_splitters(np.sort(allk[:: max(1, allk.size // 4096)]), R)
    cls, cc = [], []
    for k in shards:
        c = 2 * (spl[None, :] < k[:, None]).sum(axis=1) + (spl[None, :] == k[:, None]).any(axis=1)
        cls.append(c)
        cc.append(np.bincount(c, minlength=2 * R - 1))
    cc = np.array(cc)
    ident = [np.arange(k.size) + (r << 32) for r, k in enumerate(shards)]  # (rank, index) ids
    recv = [None] * R
    for r in range(R):
        B, delta, rcounts = exchange_plan(cc, R, r)
        if r == 0:
            recv = [np.full(int(c), -1, dtype=np.int64) for c in rcounts]
        order = np.argsort(cls[r], kind="stable")  # shard-local class-major order
        gpos = np.arange(order.size) + delta[cls[r][order]]
        d = np.searchsorted(B, gpos, side="right") - 1
        for dd in range(R):
            m = d == dd
            recv[dd][gpos[m] - B[dd]] = ident[r][order][m]
    # every element placed exactly once, each destination within its bounds
    got = np.concatenate(recv)
    assert (got >= 0).all() and np.unique(got).size == got.size == allk.size
    # same multiset per destination as the all-to-all-v path
    B = boundaries(cc, R)
    for dd in range(R):
        want = []
        for r in range(R):
            order = np.argsort(cls[r], kind="stable")
            sc = send_counts(cc, B, r)
            off = sum(sc[:dd])
            want.append(ident[r][order][off:off + sc[dd]])
        want = np.concatenate(want)
        assert np.array_equal(np.sort(recv[dd]), np.sort(want))
        # stable local sort of the class-major buffer == global (key, rank, index) order
        keys_d = np.array([shards[i >> 32][i & 0xFFFFFFFF] for i in recv[dd]], dtype=np.uint32)
        keys_w = np.array([shards[i >> 32][i & 0xFFFFFFFF] for i in want], dtype=np.uint32)
        assert np.array_equal(recv[dd][np.argsort(keys_d, kind="stable")], want[np.argsort(keys_w, kind="stable")])


@pytest.mark.parametrize("R,S", [(2, 4096), (3, 4096), (8, 4096), (8, 7)])
def test_device_splitter_indices_match_choose_splitters(R, S):
    """dist._dist_sort_peer picks sorted_samples[i*S] for i in 1..R-1 on the
    device; that is choose_splitters() on the R*S gathered samples."""
    s = np.arange(R * S, dtype=np.uint64) * np.uint64(3)
    assert np.array_equal(choose_splitters(s, R), s[np.arange(1, R) * S])


def test_dist_sort_rejects_more_than_eight_ranks(monkeypatch):
    import torch
    import torch.distributed as tdist

    from paper_0811_3448_b200 import dist as bd

    monkeypatch.setattr(tdist, "is_initialized", lambda: True)
    monkeypatch.setattr(tdist, "get_world_size", lambda group=None: 9)
    monkeypatch.setattr(tdist, "get_rank", lambda group=None: 0)
    with pytest.raises(ValueError, match="at most 8 ranks"):
        bd.dist_sort(torch.zeros(4, dtype=torch.int32), width=32)


def test_single_node_detection(monkeypatch):
    from paper_0811_3448_b200 import dist as bd

    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "4")
    assert bd._single_node(None, 4)
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "2")
    assert not bd._single_node(None, 4)


def test_peer_exchange_refused_for_cpu_tensors(monkeypatch):
    import torch
    import torch.distributed as tdist

    from paper_0811_3448_b200 import dist as bd

    monkeypatch.setattr(tdist, "is_initialized", lambda: True)
    monkeypatch.setattr(tdist, "get_world_size", lambda group=None: 2)
    monkeypatch.setattr(tdist, "get_rank", lambda group=None: 0)
    with pytest.raises(ValueError, match="peer"):
        bd.dist_sort(torch.zeros(4, dtype=torch.int32), width=32, exchange="peer")
