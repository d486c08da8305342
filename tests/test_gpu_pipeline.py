"""SortPipeline: host batches through overlapped H2D / sort / D2H streams give
exactly core.sort's output and Metrics, batch by batch."""

import numpy as np
import pytest

from paper_0811_3448_b200 import UnsignedCodec, sort
from paper_0811_3448_b200.cases import mt_words
from paper_0811_3448_b200.pipeline import SortPipeline

pytestmark = pytest.mark.gpu


def _mv(m):
    return [m.bit_extractions, m.swaps, m.recursive_calls, m.max_depth]


@pytest.mark.parametrize("dt,width", [(np.uint32, 32), (np.uint64, 64), (np.uint64, 40)])
def test_pipeline_matches_sort(cuda, dt, width):
    t = cuda
    sizes = [1 << 20, 3, 1, 0, 777_777, 1 << 20, 65_537]
    rng = np.random.default_rng(3)
    xs = [rng.integers(0, 2 ** (8 * np.dtype(dt).itemsize), s, dtype=np.uint64).astype(dt) for s in sizes]
    raw = {4: np.int32, 8: np.int64}[np.dtype(dt).itemsize]
    batches = [t.from_numpy(x.view(raw).copy()).pin_memory() for x in xs]
    outs = [t.empty_like(b).pin_memory() for b in batches]
    pipe = SortPipeline(max(sizes), batches[0].dtype, UnsignedCodec(width), slots=3)
    ms = pipe.run(batches, outs)
    for x, b, o, m in zip(xs, batches, outs, ms):
        want = x.copy()
        mw = sort(want, UnsignedCodec(width))
        assert np.array_equal(o.numpy().view(dt), want)
        assert np.array_equal(b.numpy().view(dt), x)  # inputs untouched
        assert _mv(m) == _mv(mw)


def test_pipeline_in_place_and_reuse(cuda):
    t = cuda
    pipe = SortPipeline(1 << 22, t.int32, UnsignedCodec(32), slots=2)
    for rep in range(2):
        xs = [mt_words(10 + 5 * rep + i, 1 << 22) for i in range(5)]
        batches = [t.from_numpy(x.view(np.int32).copy()).pin_memory() for x in xs]
        pipe.run(batches)
        for x, b in zip(xs, batches):
            assert np.array_equal(b.numpy().view(np.uint32), np.sort(x))
