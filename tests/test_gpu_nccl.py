"""dist_sort over a real NCCL process group, one process per GPU.

Skipped on a box with fewer than two GPUs (this run's GPU boxes have one; the
same path runs on one GPU with gloo host collectives in test_gpu_dist.py).
Each rank sorts its shard with both exchanges -- the fused peer-store kernel
(CUDA IPC mappings, regrown across calls, closed with host-blocking barriers)
and the NCCL all-to-all-v baseline -- and rank 0 checks the global order.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_WORLD_SIZE=str(world),
                      WORLD_SIZE=str(world))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from paper_0811_3448_b200.dist import _PEER_BUFFERS, dist_sort

        res = []
        for it, exchange in enumerate(["peer", "peer", "collective", "peer"]):
            rng = np.random.default_rng(100 * it + rank)
            n = (1 << 20) * (1 + it) + 101 * rank  # grows: the peer buffers regrow
            k = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
            if it == 3:
                k[: n // 2] = 0xC0FFEE  # one heavy key spread over ranks
            v = np.arange(n, dtype=np.uint32) | np.uint32(rank << 28)
            r = dist_sort(torch.from_numpy(k.view(np.int32)).to(dev), torch.from_numpy(v.view(np.int32)).to(dev),
                          width=32, exchange=exchange)
            res.append((k, v, r.keys.cpu().numpy().view(np.uint32), r.values.cpu().numpy().view(np.uint32)))
        for b in list(_PEER_BUFFERS.values()):
            b.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_dist_sort(world):
    import torch

    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (this box has {torch.cuda.device_count()})")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=500) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for it in range(len(got[0][1])):
        allk = np.concatenate([g[1][it][0] for g in got])
        allv = np.concatenate([g[1][it][1] for g in got])
        outk = np.concatenate([g[1][it][2] for g in got])
        outv = np.concatenate([g[1][it][3] for g in got])
        order = np.argsort(allk, kind="stable")
        assert np.array_equal(outk, allk[order]), it
        assert np.array_equal(outv, allv[order]), it
