"""Multi-GPU front end on ONE GPU: the fused partition + peer-store exchange.

* Emulated ranks: R shards live on cuda:0, every "rank" runs its real device
  steps (bs_sample_keys, bs_split_count, bs_split_exchange, bs_sort_from)
  with a destination table pointing at R receive buffers on the same device
  -- the kernel's stores are exactly the ones it issues to peer mappings on an
  NVSwitch node.  No kernel waits on another rank's kernel.
* Two real processes on the one GPU (gloo for the small host collectives):
  dist_sort(exchange="peer") end to end, receive buffers mapped across the
  processes with CUDA IPC (bs_ipc_*).
"""

import os
import socket
import types

import numpy as np
import pytest

from paper_0811_3448_b200 import _lib
from paper_0811_3448_b200.dist import CudaOps, choose_splitters, exchange_plan

pytestmark = pytest.mark.gpu


def _emulated(shards, vals, R, width=None, key_kind=0):
    import torch

    kb = shards[0].dtype.itemsize
    width = width or kb * 8
    ops = CudaOps(width, key_kind)
    sdt = {4: torch.int32, 8: torch.int64}[kb]
    keys = [torch.from_numpy(s.view({4: np.int32, 8: np.int64}[kb])).cuda() for s in shards]
    vt = [torch.from_numpy(v.view(np.int32)).cuda() for v in vals] if vals is not None else None
    # splitters from every shard's device samples (as dist_sort does)
    smp = torch.cat([ops.sample(k, 4096 if k.numel() else 0) for k in keys])
    ss = ops.sort_samples(smp).cpu().numpy().view({4: np.uint32, 8: np.uint64}[kb])
    spl = torch.from_numpy(choose_splitters(ss, R).view({4: np.int32, 8: np.int64}[kb])).cuda()
    per_src = []
    cc = []
    for r in range(R):
        o = CudaOps(width, key_kind)
        cc.append(o.split_count(keys[r], spl, R).cpu().numpy())
        per_src.append(o)
    cc = np.array(cc, dtype=np.int64)
    total = int(cc.sum())
    B0, _, rcounts = exchange_plan(cc, R, 0)
    recv_k = [torch.empty(max(1, int(c)), dtype=sdt, device="cuda") for c in rcounts]
    recv_v = [torch.empty(max(1, int(c)), dtype=torch.int32, device="cuda") for c in rcounts] if vals else None
    bufs = types.SimpleNamespace(
        key_table=torch.tensor([t.data_ptr() for t in recv_k], dtype=torch.int64, device="cuda"),
        val_table=torch.tensor([t.data_ptr() for t in recv_v], dtype=torch.int64, device="cuda") if vals else None)
    for r in range(R):
        B, delta, _ = exchange_plan(cc, R, r)
        per_src[r].exchange(keys[r], vt[r] if vt else None, spl, R, delta, B, bufs)
    outs = []
    for d in range(R):
        b = types.SimpleNamespace(device=recv_k[d].device, local_keys=recv_k[d].data_ptr(),
                                  local_vals=recv_v[d].data_ptr() if vals else None)
        k, v = ops.sort_from(b, int(rcounts[d]), sdt, torch.int32 if vals else None)
        outs.append((k.cpu().numpy().view(shards[0].dtype), v.cpu().numpy().view(np.uint32) if vals else None))
    assert sum(o[0].size for o in outs) == total
    return outs, B0


@pytest.mark.parametrize("R", [2, 3, 8])
@pytest.mark.parametrize("kind", ["uniform", "heavy", "sorted", "reverse"])
def test_emulated_ranks_keys(R, kind):
    rng = np.random.default_rng(R * 10 + len(kind))
    shards = []
    for r in range(R):
        n = (1 << 20) + 4099 * r
        k = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
        if kind == "heavy":
            k[rng.random(n) < 0.4] = 0xABCDEF
        shards.append(k)
    allk = np.concatenate(shards)
    if kind in ("sorted", "reverse"):
        allk = np.sort(allk) if kind == "sorted" else np.sort(allk)[::-1].copy()
        offs = np.cumsum([0] + [s.size for s in shards])
        shards = [allk[offs[r]:offs[r + 1]].copy() for r in range(R)]
    outs, B = _emulated(shards, None, R)
    got = np.concatenate([o[0] for o in outs])
    assert np.array_equal(got, np.sort(allk))
    sizes = np.array([o[0].size for o in outs])
    if kind != "heavy":
        assert sizes.max() - sizes.min() <= 0.1 * allk.size / R


@pytest.mark.parametrize("R", [2, 4])
def test_emulated_ranks_kv_stable_u64(R):
    rng = np.random.default_rng(40 + R)
    shards, vals = [], []
    for r in range(R):
        n = 300_000 + 17 * r
        shards.append(rng.integers(0, 1024, n, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15))
        vals.append((np.arange(n, dtype=np.uint32) | np.uint32(r << 28)))
    outs, _ = _emulated(shards, vals, R)
    keys = np.concatenate([o[0] for o in outs])
    got_v = np.concatenate([o[1] for o in outs])
    allk = np.concatenate(shards)
    allv = np.concatenate(vals)
    order = np.argsort(allk, kind="stable")
    assert np.array_equal(keys, allk[order])
    assert np.array_equal(got_v, allv[order])


def test_sort_from_matches_sort():
    import torch

    from paper_0811_3448_b200 import device

    rng = np.random.default_rng(5)
    for n in (0, 1, 2, 5000, 8193, 1 << 21):
        x = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
        v = np.arange(n, dtype=np.uint32)
        src = torch.from_numpy(x.view(np.int32)).cuda()
        srcv = torch.from_numpy(v.view(np.int32)).cuda()
        b = types.SimpleNamespace(device=src.device, local_keys=src.data_ptr(), local_vals=srcv.data_ptr())
        k, vv = CudaOps(32).sort_from(b, n, torch.int32, torch.int32)
        order = np.argsort(x, kind="stable")
        assert np.array_equal(k.cpu().numpy().view(np.uint32), x[order])
        assert np.array_equal(vv.cpu().numpy().view(np.uint32), v[order])
    del device


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0811_3448_b200.dist import dist_sort

        torch.cuda.set_device(0)
        res = []
        for it in range(3):  # buffers are reused (and regrown) across calls
            rng = np.random.default_rng(1000 * it + rank)
            n = (1 << 20) * (1 + it) + 333 * rank
            k = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
            v = np.arange(n, dtype=np.uint32) | np.uint32(rank << 30)
            r = dist_sort(torch.from_numpy(k.view(np.int32)).cuda(), torch.from_numpy(v.view(np.int32)).cuda(),
                          width=32, exchange="peer")
            res.append((k, v, r.keys.cpu().numpy().view(np.uint32), r.values.cpu().numpy().view(np.uint32)))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(400)
def test_two_processes_peer_exchange_one_gpu():
    import torch.multiprocessing as mp

    _lib.lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for it in range(3):
        allk = np.concatenate([g[1][it][0] for g in got])
        allv = np.concatenate([g[1][it][1] for g in got])
        outk = np.concatenate([g[1][it][2] for g in got])
        outv = np.concatenate([g[1][it][3] for g in got])
        order = np.argsort(allk, kind="stable")
        assert np.array_equal(outk, allk[order])
        assert np.array_equal(outv, allv[order])


@pytest.mark.timeout(600)
def test_bench_two_ranks_share_one_gpu():
    """bench.py's N>1 path (torchrun, dist_sort with the fused peer exchange,
    global-order check, max-over-ranks timing) with both ranks on cuda:0."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BS_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--keys-per-rank", str(1 << 22)]
    p = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=500)
    assert p.returncode == 0, p.stderr[-2000:]
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1]
    r = json.loads(line)
    assert r["n_gpus"] == 2 and r["config"]["global_batch"] == 2 << 22 and r["value"] > 0
