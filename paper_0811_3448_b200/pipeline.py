"""Host-to-host sorting of a stream of batches with the PCIe copies overlapped.

``core.sort`` on a host array is three serial steps -- copy in, sort, copy
out -- so on a B200 it runs at PCIe speed with the device idle most of the
time (a 2^28-key sort takes ~2.6 ms on the device and ~40 ms end to end).
PCIe is full duplex, so a stream of sorts can overlap batch i+1's
host-to-device copy, batch i's device sort and batch i-1's device-to-host
copy on three CUDA streams.  ``SortPipeline`` does that: every batch still
makes the whole round trip (its input is copied in, sorted with the same
``bs_sort`` call as ``core.sort``, and copied back out together with its
reference ``Metrics``), only the batches overlap each other.

This is the B200 counterpart of the reference's only batch driver -- its
benchmark loop over repeated sorts (``bench.run_plan``, bench.py:107-137) --
for host-resident data.
"""

from __future__ import annotations

from . import device
from .core import Metrics

__all__ = ["SortPipeline"]


class SortPipeline:
    """Sort pinned host batches (1-D CPU tensors of 4- or 8-byte words) in place.

    ``capacity``: the largest batch (elements); ``slots``: device buffers in
    flight (3 = one copying in, one sorting, one copying out).  ``codec`` as
    for ``core.sort`` (full-width word codecs: the fast digit sort is exact
    there; narrower widths replay the reference order with ``bs_exact_sort``).
    """

    def __init__(self, capacity: int, dtype, codec, *, device_index: int | None = None, slots: int = 3,
                 with_metrics: bool = True):
        t = device.require_cuda()
        self.t = t
        self.dev = t.device("cuda", t.cuda.current_device() if device_index is None else device_index)
        self.codec = codec
        self.dtype = dtype
        self.with_metrics = with_metrics
        probe = t.empty(0, dtype=dtype)
        self.kb = probe.element_size()
        if self.kb not in (4, 8):
            raise TypeError("SortPipeline sorts 4- or 8-byte words")
        self.key_kind = codec.gpu_spec(probe)
        if self.key_kind is None:
            raise TypeError(f"{type(codec).__name__} has no word view for {dtype}")
        self.slots = max(2, int(slots))
        raw = device._raw_dtype(self.kb)
        with t.cuda.device(self.dev):
            self.s_in, self.s_sort, self.s_out = t.cuda.Stream(), t.cuda.Stream(), t.cuda.Stream()
            self.buf = [t.empty(int(capacity), dtype=raw, device=self.dev) for _ in range(self.slots)]
            self.ctr = [t.zeros(4, dtype=t.int64, device=self.dev) for _ in range(self.slots)]
            self.stw = [t.zeros(1, dtype=t.int32, device=self.dev) for _ in range(self.slots)]
        self.ev_in = [t.cuda.Event() for _ in range(self.slots)]
        self.ev_sorted = [t.cuda.Event() for _ in range(self.slots)]
        self.ev_free = [None] * self.slots
        self.capacity = int(capacity)

    def run(self, batches, outputs=None) -> list[Metrics]:
        """Sort every batch; ``outputs[i]`` (pinned, same shape) receives batch i's
        result (default: the batch itself, in place).  Returns one Metrics per batch."""
        t = self.t
        outputs = list(batches) if outputs is None else list(outputs)
        batches = list(batches)
        if len(outputs) != len(batches):
            raise ValueError("one output per batch")
        host_ctr = t.zeros((len(batches), 4), dtype=t.int64).pin_memory()
        host_st = t.zeros(len(batches), dtype=t.int32).pin_memory()
        raw = device._raw_dtype(self.kb)
        with t.cuda.device(self.dev):
            for i, (src, dst) in enumerate(zip(batches, outputs)):
                n = src.numel()
                if n > self.capacity:
                    raise ValueError(f"batch {i} has {n} > capacity {self.capacity} elements")
                if src.element_size() != self.kb or dst.numel() != n:
                    raise ValueError("batches must match the pipeline's word size and their outputs")
                j = i % self.slots
                d = self.buf[j][:n]
                # 1. copy in (after the slot's previous batch has been copied out)
                with t.cuda.stream(self.s_in):
                    if self.ev_free[j] is not None:
                        self.s_in.wait_event(self.ev_free[j])
                    d.copy_(src.view(raw), non_blocking=True)
                    self.ev_in[j].record(self.s_in)
                # 2. sort (the same device path as core.sort)
                with t.cuda.stream(self.s_sort):
                    self.s_sort.wait_event(self.ev_in[j])
                    st = None
                    width = self.codec.width_for(src)
                    if n > 1 and width > 0:
                        c = self.ctr[j] if self.with_metrics else None
                        if width < self.kb * 8:
                            device.exact_sort_device(d, width=width, key_kind=self.key_kind, counters=c)
                            self.stw[j].zero_()
                        else:
                            st = device.sort_words_device(d, width=width, key_kind=self.key_kind, counters=c,
                                                          check=False)
                            # the status word lives in the sort stream's workspace: keep it
                            # with the slot before that stream's next sort resets it (an
                            # SM-side op: a copy here would queue behind the big D2H copies)
                            t.add(st, 0, out=self.stw[j])
                    else:
                        self.stw[j].zero_()
                        if self.with_metrics:
                            self.ctr[j].zero_()
                    self.ev_sorted[j].record(self.s_sort)
                # 3. copy out: keys, counters and the overflow status
                with t.cuda.stream(self.s_out):
                    self.s_out.wait_event(self.ev_sorted[j])
                    dst.view(raw).copy_(d, non_blocking=True)
                    if self.with_metrics:
                        host_ctr[i].copy_(self.ctr[j], non_blocking=True)
                    host_st[i:i + 1].copy_(self.stw[j], non_blocking=True)
                    ev = t.cuda.Event()
                    ev.record(self.s_out)
                    self.ev_free[j] = ev
            self.s_out.synchronize()
            self.s_sort.synchronize()
            self.s_in.synchronize()
        bad = [i for i, v in enumerate(host_st.tolist()) if v]
        if bad:
            raise device.SortOverflowError(f"device work-list overflow in batches {bad}: outputs are not sorted")
        out = []
        for i in range(len(batches)):
            m = Metrics()
            if self.with_metrics:
                m._add_counters(host_ctr[i].tolist())
            out.append(m)
        return out

    def close(self):
        self.buf = []
        self.ctr = []
        self.stw = []
