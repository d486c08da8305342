"""GPU robustness: the device overflow flag fails loudly, and concurrent sorts
on distinct streams (the reference calls its nogil kernels from pool threads,
variants.py:195-206, kernels.py:39) do not share workspaces.
"""

import threading

import numpy as np
import pytest

from paper_0811_3448_b200 import _lib, device
from paper_0811_3448_b200.cases import mt_words

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cap", [(2, 0, 0), (0, 3, 0), (0, 0, 4)])
@pytest.mark.parametrize("vb", [0, 4])
def test_forced_overflow_is_reported(cuda, cap, vb):
    """Shrunken work lists drop work; bs_sort_status must say so and the shim must raise."""
    t = cuda
    n = 1 << 23  # level-0 children exceed the local-sort size: level-1 buckets, tiles and tasks
    x = mt_words(11, n)
    k = t.from_numpy(x.view(np.int32)).cuda()
    v = t.arange(n, dtype=t.int32, device="cuda") if vb else None
    L = _lib.lib()
    L.bs_debug_capacity(*cap)
    try:
        with pytest.raises(device.SortOverflowError):
            device.sort_words_device(k, v, width=32)
    finally:
        L.bs_debug_capacity(0, 0, 0)
    # the same call without caps is clean and sorted
    k = t.from_numpy(x.view(np.int32)).cuda()
    device.sort_words_device(k, v if v is None else t.arange(n, dtype=t.int32, device="cuda"), width=32)
    assert np.array_equal(k.cpu().numpy().view(np.uint32), np.sort(x))


def test_status_clean_on_every_config_shape(cuda):
    """The status word stays 0 on the shapes the planner finds hardest (ties, skew, tiny)."""
    t = cuda
    rng = np.random.default_rng(5)
    inputs = [
        np.zeros(1 << 18, np.uint32),
        rng.integers(0, 3, 1 << 20).astype(np.uint32),
        (rng.zipf(1.1, 1 << 20) & 0xFFFFFFFF).astype(np.uint32),
        np.arange(1 << 20, dtype=np.uint32)[::-1].copy(),
        rng.integers(0, 1 << 63, 1 << 19, dtype=np.uint64),
    ]
    for x in inputs:
        k = t.from_numpy(x.view(np.int32 if x.itemsize == 4 else np.int64)).cuda()
        st = device.sort_words_device(k, width=x.itemsize * 8, check=False)
        device.check_status(st)
        assert np.array_equal(k.cpu().numpy().view(x.dtype), np.sort(x))


def test_concurrent_sorts_on_distinct_streams(cuda):
    """Four threads, each on its own stream, sort different arrays at once."""
    t = cuda
    n = 3 << 20
    datas = [mt_words(100 + i, n) for i in range(4)]
    outs = [None] * 4
    errs = []
    start = threading.Barrier(4)

    def work(i):
        try:
            s = t.cuda.Stream()
            with t.cuda.stream(s):
                k = t.from_numpy(datas[i].view(np.int32)).cuda()
                start.wait()
                for _ in range(3):
                    k2 = k.clone()
                    device.sort_words_device(k2, width=32)
                outs[i] = k2.cpu().numpy().view(np.uint32)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    assert not errs, errs
    for i in range(4):
        assert np.array_equal(outs[i], np.sort(datas[i])), i


def test_workspace_cache_is_per_stream(cuda):
    t = cuda
    s1, s2 = t.cuda.Stream(), t.cuda.Stream()
    a = device.workspaces.get(1 << 20, "cuda", s1)
    b = device.workspaces.get(1 << 20, "cuda", s2)
    assert a.data_ptr() != b.data_ptr()
    assert device.workspaces.get(1 << 10, "cuda", s1).data_ptr() == a.data_ptr()
