"""Multi-GPU front end: one process per GPU, range partition + a fused peer-memory exchange.

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
4. **Data exchange** -- the product path (``exchange="peer"``) fuses steps 2
   and 4: once every rank's class counts are known, every element's position
   in the global class-major order is too, so ``bs_split_exchange`` stores
   each element straight into its destination rank's receive buffer over
   NVLink / NVSwitch peer memory (buffers mapped once with CUDA IPC and
   reused), one kernel instead of partition -> send buffer -> all-to-all-v.
   ``exchange="collective"`` keeps the partition + ``all_to_all_single``
   (NCCL) form as the baseline and for the CPU (gloo) tests.
5. **Local sort** -- each receive buffer holds its global positions
   [B[d], B[d+1]) in class-major, source-rank order and is sorted by the
   single-GPU sort (stable; ``bs_sort_from`` writes the result to a fresh
   tensor, the receive buffer is its ping-pong copy), so rank r ends up owning
   the r-th contiguous slice of the global sorted order.

The per-rank device steps go through a ``LocalOps`` object; the product uses
:class:`CudaOps` (the C ABI).  The host logic (splitters, tie division,
split sizes) is plain Python so it can be exercised with gloo on CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, device

__all__ = ["CudaOps", "DistResult", "PeerBuffers", "choose_splitters", "boundaries", "send_counts",
           "exchange_plan", "dist_sort", "PeerUnavailable"]


@dataclass
class DistResult:
    keys: object  # this rank's slice of the globally sorted order
    values: object | None
    send_counts: list[int]
    recv_counts: list[int]
    exchange: str = ""  # the data exchange that ran: "peer", "collective" (or "" for one rank)


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

    # ---- fused peer exchange (exchange="peer") ----
    def split_count(self, keys, splitters, nranks: int):
        """Class counts of this shard (device uint64 as int64); tile offsets stay in self._split_ws."""
        t = device.require_cuda()
        L = _lib.lib()
        n = keys.numel()
        kb = keys.element_size()
        counts = t.zeros(2 * nranks - 1, dtype=t.int64, device=keys.device)
        need = L.bs_split_workspace_bytes(n, kb, 0, nranks)
        ws = getattr(self, "_split_ws", None)
        if ws is None or ws.numel() < need or ws.device != keys.device:
            ws = self._split_ws = t.empty(need, dtype=t.uint8, device=keys.device)
        with t.cuda.device(keys.device):
            rc = L.bs_split_count(keys.data_ptr(), n, kb, self.width, self.key_kind, splitters.data_ptr(), nranks,
                                  counts.data_ptr(), ws.data_ptr(), ws.numel(), device.stream_ptr(keys.device))
        _lib.check(rc)
        # the workspace now holds THIS shard's per-tile class offsets, which exchange() reads
        self._counted = (keys.data_ptr(), n, splitters.data_ptr(), nranks)
        return counts

    def exchange(self, keys, values, splitters, nranks: int, delta: np.ndarray, bounds: np.ndarray, bufs):
        """Store every element into its destination's receive buffer (bs_split_exchange).

        Must follow ``split_count`` of the same shard with the same splitters on this object
        (the kernel reads the tile offsets that pass left in the workspace)."""
        t = device.require_cuda()
        L = _lib.lib()
        dev = keys.device
        if getattr(self, "_counted", None) != (keys.data_ptr(), keys.numel(), splitters.data_ptr(), nranks):
            raise ValueError("exchange() must follow split_count() of the same shard and splitters on this CudaOps "
                             "(one CudaOps per source rank)")
        d_delta = t.from_numpy(np.ascontiguousarray(delta, dtype=np.int64)).to(dev, non_blocking=True)
        d_bounds = t.from_numpy(np.ascontiguousarray(bounds, dtype=np.int64)).to(dev, non_blocking=True)
        ws = self._split_ws
        with t.cuda.device(dev):
            rc = L.bs_split_exchange(keys.data_ptr(), values.data_ptr() if values is not None else None,
                                     keys.numel(), keys.element_size(),
                                     values.element_size() if values is not None else 0, self.width,
                                     self.key_kind, splitters.data_ptr(), nranks, d_delta.data_ptr(),
                                     d_bounds.data_ptr(), bufs.key_table.data_ptr(),
                                     bufs.val_table.data_ptr() if values is not None else None,
                                     ws.data_ptr(), ws.numel(), device.stream_ptr(dev))
        _lib.check(rc)

    def sort_from(self, bufs, count: int, key_dtype, val_dtype):
        """Sort this rank's receive buffer into fresh tensors (bs_sort_from)."""
        t = device.require_cuda()
        L = _lib.lib()
        dev = bufs.device
        out_k = t.empty(count, dtype=key_dtype, device=dev)
        out_v = t.empty(count, dtype=val_dtype, device=dev) if val_dtype is not None else None
        kb = out_k.element_size()
        vb = out_v.element_size() if out_v is not None else 0
        ws = device.workspaces.get(L.bs_sort_from_workspace_bytes(count, kb, vb), dev)
        with t.cuda.device(dev):
            rc = L.bs_sort_from(bufs.local_keys, bufs.local_vals if vb else None, out_k.data_ptr(),
                                out_v.data_ptr() if out_v is not None else None, count, kb, vb, self.width, 0,
                                self.key_kind, ws.data_ptr(), ws.numel(), device.stream_ptr(dev))
            _lib.check(rc)
            if count > 1:
                status = t.empty(1, dtype=t.int32, device=dev)
                _lib.check(L.bs_sort_status(ws.data_ptr(), status.data_ptr(), device.stream_ptr(dev)))
                device.check_status(status)
        return out_k, out_v


class PeerUnavailable(RuntimeError):
    """The CUDA IPC peer mappings could not be set up (raised on EVERY rank of the group)."""


class PeerBuffers:
    """Per-rank receive buffers mapped into every rank's address space (CUDA IPC).

    One allocation per rank holds ``cap`` keys (and ``cap`` values); the
    handles are all-gathered once and every peer's buffer is opened, so the
    exchange kernel can store to ``key_table[d]`` for any destination d.  The
    buffers are reused across calls and regrown collectively (every rank
    derives the same required capacity from the all-gathered class counts).
    """

    def __init__(self, group, dev):
        self.group = group
        self.device = dev
        self.cap = 0
        self.kb = self.vb = 0
        self._local = None
        self._peers = []
        self.key_table = self.val_table = None
        self.local_keys = self.local_vals = None

    def ensure(self, cap: int, kb: int, vb: int) -> "PeerBuffers":
        import ctypes

        import torch

        if cap <= self.cap and kb == self.kb and vb == self.vb:
            return self
        self.close()
        L = _lib.lib()
        cap = max(1024, int(cap * 1.125) + 1024)
        voff = (cap * kb + 255) // 256 * 256
        nbytes = voff + cap * vb
        R = _world(self.group)
        me = _rank(self.group)
        hb = int(L.bs_ipc_handle_bytes())
        handle = (ctypes.c_ubyte * hb)()
        ptr = ctypes.c_void_p()
        # Every step that can fail on ONE rank (allocation, opening a peer's
        # handle) is followed by an all-gathered verdict, so all ranks take the
        # same exit: a rank that raised alone would leave the others waiting in
        # the next collective.
        why = ""
        try:
            with torch.cuda.device(self.device):
                _lib.check(L.bs_ipc_alloc(nbytes, ctypes.byref(ptr), handle))
            self._local = ptr.value
        except Exception as e:  # noqa: BLE001 - reported collectively below
            why = f"rank {me}: bs_ipc_alloc: {e}"
        msg = np.zeros(hb + 1, dtype=np.uint8)
        msg[:hb] = np.frombuffer(bytes(handle), dtype=np.uint8)
        msg[hb] = 0 if why else 1
        allmsg = _all_gather_np(msg, self.group, self.device)
        handles = allmsg[:, :hb]
        bases = []
        if allmsg[:, hb].all():
            try:
                with torch.cuda.device(self.device):
                    for r in range(R):
                        if r == me:
                            bases.append(self._local)
                            continue
                        p = ctypes.c_void_p()
                        _lib.check(L.bs_ipc_open(handles[r].tobytes(), ctypes.byref(p)))
                        self._peers.append(p.value)
                        bases.append(p.value)
            except Exception as e:  # noqa: BLE001
                why = f"rank {me}: bs_ipc_open: {e}"
        elif not why:
            why = "a peer could not allocate its receive buffer"
        verdict = _all_gather_np(np.array([0 if why else 1], dtype=np.uint8), self.group, self.device)
        if not verdict.all():
            self._abort()
            bad = [int(r) for r in np.nonzero(verdict[:, 0] == 0)[0]]
            raise PeerUnavailable(why or f"peer mapping failed on rank(s) {bad}")
        self.key_table = torch.tensor(bases, dtype=torch.int64, device=self.device)
        self.val_table = torch.tensor([b + voff for b in bases], dtype=torch.int64, device=self.device)
        self.local_keys = self._local
        self.local_vals = self._local + voff
        self.cap, self.kb, self.vb = cap, kb, vb
        return self

    def _abort(self) -> None:
        """Collective clean-up after a failed ``ensure``: every rank runs both barriers."""
        import torch

        L = _lib.lib()
        torch.cuda.synchronize(self.device)
        _host_barrier(self.group, self.device)
        for p in self._peers:
            L.bs_ipc_close(p)
        _host_barrier(self.group, self.device)
        if self._local is not None:
            L.bs_ipc_free(self._local)
        self._local = None
        self._peers = []
        self.cap = 0

    def close(self) -> None:
        if self._local is None:
            return
        import torch

        L = _lib.lib()
        torch.cuda.synchronize(self.device)
        _host_barrier(self.group, self.device)  # nobody still stores into or reads from these buffers
        for p in self._peers:
            _lib.check(L.bs_ipc_close(p))
        # every peer has closed its mapping of our buffer (host-blocking: cudaFree
        # of an exported region before the importers close it is undefined)
        _host_barrier(self.group, self.device)
        _lib.check(L.bs_ipc_free(self._local))
        self._local = None
        self._peers = []
        self.cap = 0


_PEER_BUFFERS: dict = {}
_NO_PEER: set = set()  # groups whose peer mappings failed once: exchange="auto" stays collective


def _peer_buffers(group, dev) -> PeerBuffers:
    key = (id(group), str(dev))
    b = _PEER_BUFFERS.get(key)
    if b is None:
        b = _PEER_BUFFERS[key] = PeerBuffers(group, dev)
    return b


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


def exchange_plan(class_counts: np.ndarray, nranks: int, rank: int):
    """Host side of the fused exchange for source ``rank``.

    Returns (bounds B[0..R], delta[2R-1], recv_counts[R]): destination d owns
    global class-major positions [B[d], B[d+1]); this rank's shard-local
    class-major position p of a class-c element maps to the global position
    p + delta[c] (global order: class, then source rank, then shard index --
    the order ``send_counts`` / the all-to-all path produce).
    """
    cc = np.asarray(class_counts, dtype=np.int64)
    B = boundaries(cc, nranks)
    totals = cc.sum(axis=0)
    cstart = np.concatenate([[0], np.cumsum(totals)])[:-1]
    gbase = cstart + cc[:rank].sum(axis=0)
    lbase = np.concatenate([[0], np.cumsum(cc[rank])])[:-1]
    return B, (gbase - lbase).astype(np.int64), np.diff(B).astype(np.int64)


def _world(group) -> int:
    import torch.distributed as dist

    return dist.get_world_size(group) if dist.is_initialized() else 1


def _rank(group) -> int:
    import torch.distributed as dist

    return dist.get_rank(group) if dist.is_initialized() else 0


def _on_device(group) -> bool:
    import torch.distributed as dist

    return dist.get_backend(group) == "nccl"


def _all_gather_np(a: np.ndarray, group, dev) -> np.ndarray:
    """All-gather a small host array over ``group`` -> [R, *a.shape] (device tensors for NCCL)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(a).copy())
    if _on_device(group):
        t = t.to(dev)
    out = [torch.empty_like(t) for _ in range(_world(group))]
    dist.all_gather(out, t, group=group)
    return np.stack([o.cpu().numpy() for o in out])


def _barrier(group, dev) -> None:
    """Order every rank's queued device work before what follows on any rank."""
    import torch
    import torch.distributed as dist

    if _on_device(group):  # stream-ordered: a one-element all-reduce on the current stream
        dist.all_reduce(torch.zeros(1, device=dev), group=group)
    else:
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)


def _host_barrier(group, dev) -> None:
    """Barrier that returns only when every rank has reached it AND its queued device work is done."""
    import torch
    import torch.distributed as dist

    torch.cuda.synchronize(dev)
    if _on_device(group):
        dist.all_reduce(torch.zeros(1, device=dev), group=group)
        torch.cuda.synchronize(dev)  # the NCCL all-reduce itself only orders the stream
    else:
        dist.barrier(group=group)


# Splitter samples per rank: the destination loads deviate from N/R by about
# sqrt(R / (4 * S)) of N/R per boundary, so 65536 keeps them within ~0.5 %
# at R = 8 (4096 gave ~2-4 % on cfg5); sorting R*S samples costs ~0.1 ms.
SAMPLES_PER_RANK = 65536

MAX_RANKS = 8  # the split kernels classify into 2R-1 <= 15 classes (16-wide tile rows)


def _single_node(group, R: int) -> bool:
    """True when every rank of ``group`` runs on this host (CUDA IPC peer mappings need it)."""
    import os
    import socket

    lws, ws = os.environ.get("LOCAL_WORLD_SIZE"), os.environ.get("WORLD_SIZE")
    if lws is not None and ws is not None and int(ws) == R:
        return int(lws) == int(ws)
    import torch.distributed as dist

    names = [None] * R
    dist.all_gather_object(names, socket.gethostname(), group=group)
    return len(set(names)) == 1


def dist_sort(keys, values=None, *, width: int, key_kind: int = _lib.BS_KEY_UNSIGNED, ops=None, group=None,
              samples_per_rank: int = SAMPLES_PER_RANK, exchange: str = "auto", marks: list | None = None) -> DistResult:
    """Globally sort the shards held by all ranks of ``group``.

    ``keys`` (and ``values``) are this rank's contiguous 1-D tensors (CUDA for
    the product path).  Returns this rank's slice of the global order; the
    concatenation over ranks 0..R-1 is the sorted whole.  ``exchange``:
    "peer" (fused partition + peer-memory stores, the product path for CUDA
    tensors on one node), "collective" (partition + all-to-all-v), or "auto"
    ("peer" for CUDA tensors when every rank is on this node, else
    "collective").  ``marks`` (instrumentation): a list that receives
    ``(phase, cuda.Event)`` pairs recorded on the current stream at the phase
    boundaries of the peer path (bench.py's per-phase roofline).

    Scope: one NVLink/NVSwitch node of at most ``MAX_RANKS`` (8) GPUs -- the
    B200 HGX node the fused exchange is built for.  Larger groups raise
    ``ValueError`` up front; "peer" across nodes raises ``ValueError`` (CUDA
    IPC mappings do not cross hosts).
    """
    import torch
    import torch.distributed as dist

    ops = ops or CudaOps(width, key_kind)
    if exchange not in ("auto", "peer", "collective"):
        raise ValueError(f"unknown exchange {exchange!r}")
    R = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if R > MAX_RANKS:
        raise ValueError(f"dist_sort supports at most {MAX_RANKS} ranks (one NVSwitch node), got {R}")
    auto = exchange == "auto"
    if exchange != "collective" and R > 1:
        cuda_path = isinstance(ops, CudaOps) and getattr(keys, "is_cuda", False)
        one_node = cuda_path and _single_node(group, R)
        if exchange == "auto":
            exchange = "peer" if one_node and id(group) not in _NO_PEER else "collective"
        elif not one_node:
            raise ValueError("exchange='peer' needs CUDA tensors and every rank on one node (CUDA IPC)")
    if R == 1:
        k, v = ops.sort(keys, values)
        return DistResult(k, v, [keys.numel()], [keys.numel()])
    dev = keys.device
    if exchange == "peer":
        try:
            res = _dist_sort_peer(keys, values, ops, group, R, rank, samples_per_rank, marks)
            res.exchange = "peer"
            return res
        except PeerUnavailable as e:
            # raised on every rank (PeerBuffers.ensure agrees collectively), before any data moved
            if not auto:
                raise
            import warnings

            warnings.warn(f"dist_sort: peer-memory exchange unavailable ({e}); using the collective exchange")
            _NO_PEER.add(id(group))
            if marks is not None:
                del marks[:]
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
    return DistResult(recv_k, recv_v, scounts, rcounts, "collective")


def _all_gather_dev(t, group):
    """All-gather a small device tensor -> [R, *t.shape] on the same device (one collective)."""
    import torch
    import torch.distributed as dist

    R = _world(group)
    if _on_device(group):
        out = torch.empty((R,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out
    parts = [torch.empty_like(t) for _ in range(R)]
    dist.all_gather(parts, t.contiguous(), group=group)
    return torch.stack(parts)


def _dist_sort_peer(keys, values, ops, group, R: int, rank: int, S: int, marks=None) -> DistResult:
    """dist_sort with the fused partition + peer-store exchange (one host sync per call)."""
    import torch

    def mark(name):
        if marks is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            marks.append((name, ev))

    dev = keys.device
    mark("start")
    # 1. splitters on the device: S normalised samples per rank (an empty shard
    # contributes the maximum word), all-gathered, sorted, quantiles i*S
    if keys.numel():
        smp = ops.sample(keys, S)
    else:
        smp = torch.full((S,), -1, dtype=keys.dtype, device=dev)
    ssorted = ops.sort_samples(_all_gather_dev(smp, group).reshape(-1))
    splitters = ssorted[torch.arange(1, R, device=dev) * S].contiguous()  # == choose_splitters
    mark("splitters")
    # 2+3. class counts of every shard; the one host read also orders this
    # rank's previous local sort (which reads its receive buffer) before the
    # all-gather completes anywhere, so no peer overwrites a buffer in use
    counts = ops.split_count(keys, splitters, R)
    mark("class_count")
    cc = _all_gather_dev(counts, group).cpu().numpy().astype(np.int64)
    B, delta, rcounts = exchange_plan(cc, R, rank)
    kb = keys.element_size()
    vb = values.element_size() if values is not None else 0
    bufs = _peer_buffers(group, dev).ensure(int(rcounts.max()), kb, vb)
    # 4. fused partition + peer stores, then every rank's stores land
    mark("plan")
    ops.exchange(keys, values, splitters, R, delta, B, bufs)
    mark("exchange")
    _barrier(group, dev)
    mark("barrier")
    # 5. local sort out of the receive buffer
    out_k, out_v = ops.sort_from(bufs, int(rcounts[rank]), keys.dtype, values.dtype if values is not None else None)
    mark("local_sort")
    scounts = send_counts(cc, B, rank)
    return DistResult(out_k, out_v, scounts, [send_counts(cc, B, src)[rank] for src in range(R)])


def _np_signed(itemsize: int):
    return {4: np.int32, 8: np.int64}[itemsize]


def _to_unsigned_np(t) -> np.ndarray:
    a = t.cpu().numpy()
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])
