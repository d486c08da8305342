"""Multi-GPU front end: one process per GPU, range partition + one all-to-all-v.

Replaces the reference's bucket parallelism (``variants.sort_parallel``,
``variants.py:162-229``: a serial top-bit pre-partition on the main thread,
then a thread pool over disjoint buckets) with the distributed form the paper
sketches (``PAPER.md:479``) and SURVEY §8e specifies:

1. **Splitters** -- every rank samples its shard (``bs_sample_keys``, encoded
   and normalised keys), the samples are all-gathered and sorted on the
   device, and R-1 splitters are taken at the sample quantiles.  Sampling
   adapts to skew (Zipf, low-entropy, sorted/reverse inputs) where a fixed
   top-bit split would not.
2. **Destination partition** -- one stable device pass
   (``bs_split_by_splitters``) orders the shard into 2R-1 classes: keys
   strictly between splitters, and keys *equal* to each splitter.
3. **Count exchange** -- the class counts are all-gathered; keys equal to a
   splitter may be divided among neighbouring ranks by count, in global
   (rank, local index) order, so destination loads stay balanced even when
   one key value holds a large share of the data, and a stable sort stays
   stable across ranks.
4. **Data exchange** -- ``all_to_all_single`` (NCCL over NVLink/NVSwitch on
   B200; gloo in the CPU tests); every destination's data is one contiguous
   run of the partitioned shard.
5. **Local sort** -- the received runs arrive in source-rank order and are
   sorted by the single-GPU ``bs_sort`` (stable), so rank r ends up owning the
   r-th contiguous slice of the global sorted order.

The per-rank device steps go through a ``LocalOps`` object; the product uses
:class:`CudaOps` (the C ABI).  The host logic (splitters, tie division,
split sizes) is plain Python so it can be exercised with gloo on CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, device

__all__ = ["CudaOps", "DistResult", "choose_splitters", "boundaries", "send_counts", "dist_sort"]


@dataclass
class DistResult:
    keys: object  # this rank's slice of the globally sorted order
    values: object | None
    send_counts: list[int]
    recv_counts: list[int]


class CudaOps:
    """Per-rank device steps through ``libbinarsort_b200.so``."""

    def __init__(self, width: int, key_kind: int = _lib.BS_KEY_UNSIGNED):
        self.width = width
        self.key_kind = key_kind

    def sample(self, keys, count: int):
        t = device.require_cuda()
        L = _lib.lib()
        out = t.empty(count, dtype=keys.dtype, device=keys.device)
        if keys.numel() == 0 or count == 0:
            return out[:0]
        with t.cuda.device(keys.device):
            rc = L.bs_sample_keys(keys.data_ptr(), keys.numel(), keys.element_size(), self.width, self.key_kind,
                                  count, out.data_ptr(), device.stream_ptr(keys.device))
        _lib.check(rc)
        return out

    def sort_samples(self, samples):
        """Sort encoded/normalised sample words as plain unsigned words."""
        s = samples.contiguous().clone()
        if s.numel() > 1:
            device.sort_words_device(s, width=s.element_size() * 8)
        return s

    def split(self, keys, values, splitters, nranks: int):
        t = device.require_cuda()
        L = _lib.lib()
        n = keys.numel()
        kb = keys.element_size()
        vb = values.element_size() if values is not None else 0
        out_k = t.empty_like(keys)
        out_v = t.empty_like(values) if values is not None else None
        counts = t.zeros(2 * nranks - 1, dtype=t.int64, device=keys.device)
        ws = device.workspaces.get(L.bs_split_workspace_bytes(n, kb, vb, nranks), keys.device)
        spl = splitters.contiguous()
        with t.cuda.device(keys.device):
            rc = L.bs_split_by_splitters(keys.data_ptr(), values.data_ptr() if values is not None else None, n, kb,
                                         vb, self.width, self.key_kind, spl.data_ptr(), nranks, out_k.data_ptr(),
                                         out_v.data_ptr() if out_v is not None else None, counts.data_ptr(),
                                         ws.data_ptr(), ws.numel(), device.stream_ptr(keys.device))
        _lib.check(rc)
        return out_k, out_v, counts

    def sort(self, keys, values):
        if keys.numel() > 1:
            device.sort_words_device(keys, values, width=self.width, key_kind=self.key_kind)
        return keys, values


def choose_splitters(sorted_samples: np.ndarray, nranks: int) -> np.ndarray:
    """R-1 splitters at the quantiles i*S/R of the sorted samples."""
    s = len(sorted_samples)
    if nranks <= 1 or s == 0:
        return sorted_samples[:0]
    idx = [min(s - 1, (i * s) // nranks) for i in range(1, nranks)]
    return sorted_samples[idx]


def boundaries(class_counts: np.ndarray, nranks: int) -> np.ndarray:
    """Destination boundaries B[0..R] in the global class order.

    ``class_counts`` is [R_src, 2R-1] (rows = source ranks).  The global order
    is class-major, then source rank, then local index.  Destination d owns
    global positions [B[d], B[d+1]).  A boundary may cut a tie class (odd
    class: keys equal to a splitter -- all equal, any cut keeps the order) but
    never an even class (keys strictly between splitters, not yet sorted), so
    B[d] is d*N/R where that lands in a tie class, else the nearer end of the
    even class it lands in.  One heavy key value can therefore be spread over
    several destinations, in global (rank, index) order.
    """
    totals = class_counts.sum(axis=0).astype(np.int64)
    n = int(totals.sum())
    starts = np.concatenate([[0], np.cumsum(totals)])
    B = np.zeros(nranks + 1, dtype=np.int64)
    B[nranks] = n
    for d in range(1, nranks):
        t = (d * n) // nranks
        c = int(np.searchsorted(starts, t, side="right")) - 1
        c = min(c, len(totals) - 1)
        if c % 2 == 1:
            b = t
        else:
            lo, hi = int(starts[c]), int(starts[c + 1])
            b = lo if (t - lo) <= (hi - t) else hi
        B[d] = max(b, B[d - 1])
    return B


def send_counts(class_counts: np.ndarray, B: np.ndarray, rank: int) -> list[int]:
    """Elements source ``rank`` sends to each destination.

    The source's shard is ordered by class, and within each class its block is
    one contiguous interval of the global order, so what it sends to each
    destination is one contiguous run of its partitioned shard.
    """
    nranks = len(B) - 1
    totals = class_counts.sum(axis=0).astype(np.int64)
    starts = np.concatenate([[0], np.cumsum(totals)])
    out = [0] * nranks
    for c in range(class_counts.shape[1]):
        mine = int(class_counts[rank, c])
        if mine == 0:
            continue
        gs = int(starts[c]) + int(class_counts[:rank, c].sum())
        ge = gs + mine
        for d in range(nranks):
            lo, hi = max(gs, int(B[d])), min(ge, int(B[d + 1]))
            if hi > lo:
                out[d] += hi - lo
    return out


def dist_sort(keys, values=None, *, width: int, key_kind: int = _lib.BS_KEY_UNSIGNED, ops=None, group=None,
              samples_per_rank: int = 4096) -> DistResult:
    """Globally sort the shards held by all ranks of ``group``.

    ``keys`` (and ``values``) are this rank's contiguous 1-D tensors (CUDA for
    the product path).  Returns this rank's slice of the global order; the
    concatenation over ranks 0..R-1 is the sorted whole.
    """
    import torch
    import torch.distributed as dist

    ops = ops or CudaOps(width, key_kind)
    R = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if R == 1:
        k, v = ops.sort(keys, values)
        return DistResult(k, v, [keys.numel()], [keys.numel()])
    dev = keys.device
    # 1. splitters from gathered samples
    smp = ops.sample(keys, samples_per_rank if keys.numel() else 0)
    cnt = torch.tensor([smp.numel()], dtype=torch.int64, device=dev)
    all_cnt = [torch.zeros_like(cnt) for _ in range(R)]
    dist.all_gather(all_cnt, cnt, group=group)
    m = max(int(c.item()) for c in all_cnt)
    pad = torch.zeros(m, dtype=keys.dtype, device=dev)
    pad[:smp.numel()] = smp
    gathered = [torch.empty_like(pad) for _ in range(R)]
    dist.all_gather(gathered, pad, group=group)
    allsmp = torch.cat([g[:int(c.item())] for g, c in zip(gathered, all_cnt)])
    ssorted = ops.sort_samples(allsmp)
    spl_host = choose_splitters(_to_unsigned_np(ssorted), R)
    splitters = torch.from_numpy(spl_host.view(_np_signed(keys.element_size()))).to(dev)
    # 2. destination partition
    send_k, send_v, class_counts = ops.split(keys, values, splitters, R)
    # 3. count exchange + tie division
    all_cc = [torch.zeros_like(class_counts) for _ in range(R)]
    dist.all_gather(all_cc, class_counts, group=group)
    cc = np.stack([c.cpu().numpy() for c in all_cc]).astype(np.int64)
    B = boundaries(cc, R)
    scounts = send_counts(cc, B, rank)
    rcounts = [send_counts(cc, B, src)[rank] for src in range(R)]
    # 4. all-to-all-v
    recv_k = torch.empty(sum(rcounts), dtype=keys.dtype, device=dev)
    dist.all_to_all_single(recv_k, send_k, rcounts, scounts, group=group)
    recv_v = None
    if values is not None:
        recv_v = torch.empty(sum(rcounts), dtype=values.dtype, device=dev)
        dist.all_to_all_single(recv_v, send_v, rcounts, scounts, group=group)
    # 5. local (stable) sort; sources arrive in rank order
    recv_k, recv_v = ops.sort(recv_k, recv_v)
    return DistResult(recv_k, recv_v, scounts, rcounts)


def _np_signed(itemsize: int):
    return {4: np.int32, 8: np.int64}[itemsize]


def _to_unsigned_np(t) -> np.ndarray:
    a = t.cpu().numpy()
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])
