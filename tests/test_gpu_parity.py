"""GPU parity: the sm_100a CUDA path (through the C ABI) vs the reference.

Oracles: tests/golden/golden.json (outputs of the reference package itself,
tests/golden/make_golden.py) and the C oracle oracle/binarsort_oracle.c
(pinned to the same golden vectors in test_oracle_golden.py).  Keys-only
output must be bit-exact; key-value output must be the stable order (equal to
the reference's sort of packed (key << 32 | index) words).
"""

import hashlib

import numpy as np
import pytest

import paper_0811_3448_b200 as bs
from paper_0811_3448_b200 import cases, device, kernels
from paper_0811_3448_b200.core import Metrics, SortRange
from paper_0811_3448_b200.keys import Float64Codec, SignedCodec, UnsignedCodec

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def mvec(m):
    return [m.bit_extractions, m.swaps, m.recursive_calls, m.max_depth]


# --------------------------------------------------------------------------
# reference known answers
# --------------------------------------------------------------------------

def test_nybble_worked_example(cuda, golden):
    g = golden["nybble_sort"]
    seq = list(g["input"])
    m = bs.sort(seq, UnsignedCodec(4))
    assert seq == g["output"] and mvec(m) == g["metrics"]


def test_paper_partitions_exact(cuda, golden):
    for p in golden["partitions_w4"]:
        seq = list(p["input"])
        mm = Metrics()
        r = bs.partition(seq, SortRange(0, len(seq) - 1, p["pos"]), UnsignedCodec(4), mm)
        assert seq == p["output"] and r.split == p["split"] and r.pass_through == p["pass_through"]
        assert mm.bit_extractions == p["extractions"] and mm.swaps == p["swaps"]


def test_tagged_swap_order(cuda, golden):
    # tests/test_core.py:65-71: tags e,b,d,c,a -- the exact unstable movement
    g = golden["tagged_partition"]
    keys = list(g["keys"])
    tags = np.arange(len(keys), dtype=np.uint32)
    r = bs.partition(keys, SortRange(0, len(keys) - 1, 0), UnsignedCodec(4), Metrics(), values=tags)
    assert [g["tags"][i] for i in tags] == g["out_tags"] and r.split == g["split"]


def test_zero_one_depth(cuda, golden):
    seq = [0, 1]
    assert mvec(bs.sort(seq, UnsignedCodec(8))) == golden["zero_one_w8"]


def test_kernel_sorts_with_counters(cuda, golden):
    rng = {32: np.random.default_rng(21), 64: np.random.default_rng(21)}
    for g in golden["kernel_sorts"]:
        w, size = g["width"], g["size"]
        dt = np.uint32 if w == 32 else np.uint64
        a = rng[w].integers(0, 2 ** w, size, dtype=np.uint64).astype(dt)
        c = kernels.new_counters()
        if size > 1:
            kernels.sort_words(a, 0, size - 1, 0, w, False, 0, 0, False, c, 1)
        assert sha(a) == g["output_sha"], (w, size)
        assert c.tolist() == g["counters"], (w, size)


def test_kernel_partitions_exact(cuda, golden):
    rng = np.random.default_rng(5)
    for g in golden["kernel_partitions"]["cases"]:
        n = int(rng.integers(1, 3000))
        w = int(rng.choice([8, 16, 32]))
        pos = int(rng.integers(0, w))
        a = rng.integers(0, 2 ** w, n, dtype=np.uint64).astype(np.uint32)
        c = kernels.new_counters()
        split = kernels.partition_words(a, 0, n - 1, pos, w, c)
        assert sha(a) == g["output_sha"] and split == g["split"] and c.tolist() == g["counters"]


def test_cfg1_bit_exact_with_metrics(cuda, golden):
    g = golden["cfg1"]
    x = cases.config1()
    m = bs.sort(x, UnsignedCodec(32))
    assert sha(x) == g["output_sha"] and mvec(m) == g["metrics"]


# --------------------------------------------------------------------------
# differential vs the C oracle (reference restatement)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("dt,w", [(np.uint32, 32), (np.uint64, 64), (np.uint32, 20), (np.uint64, 40)])
def test_random_sizes_vs_oracle(cuda, oracle_lib, dt, w):
    rng = np.random.default_rng(w)
    for n in (2, 3, 31, 257, 4097, 8191, 8192, 8193, 20000, 100003, 1 << 20):
        x = rng.integers(0, 2 ** w, n, dtype=np.uint64).astype(dt)
        want = x.copy()
        wc = oracle_lib.sort(want, w)
        got = x.copy()
        m = bs.sort(got, UnsignedCodec(w))
        assert np.array_equal(got, want), (w, n)
        assert mvec(m) == wc.tolist(), (w, n)


def test_low_width_words_keep_high_bits(cuda):
    # UnsignedCodec(32) on u64 words orders by the low 32 bits (keys.py:175-178)
    rng = np.random.default_rng(3)
    x = rng.integers(0, 2 ** 64, 50000, dtype=np.uint64)
    got = x.copy()
    bs.sort(got, UnsignedCodec(32))
    low = got & np.uint64(0xFFFFFFFF)
    assert np.all(low[1:] >= low[:-1])
    assert np.array_equal(np.sort(got), np.sort(x))


def test_subrange_start_pos_matches_oracle(cuda, oracle_lib):
    # sort_words(arr, lo, up, pos, ...) as called by sort_parallel (variants.py:195-200)
    rng = np.random.default_rng(9)
    for pos, depth in ((3, 4), (8, 9), (17, 2)):
        x = rng.integers(0, 2 ** 32, 30000, dtype=np.uint64).astype(np.uint32)
        lo, up = 100, 25000
        a, b = x.copy(), x.copy()
        ca, cb = oracle_lib.new_counters(), kernels.new_counters()
        oracle_lib.sort_words(a, lo, up, pos, 32, False, 0, 0, False, ca, depth)
        kernels.sort_words(b, lo, up, pos, 32, False, 0, 0, False, cb, depth)
        assert np.array_equal(a[:lo], b[:lo]) and np.array_equal(a[up + 1:], b[up + 1:])
        # keys differing above `pos` are ties for this call: compare as multisets per bit-suffix order
        mask = np.uint32((1 << (32 - pos)) - 1)
        assert np.array_equal(a[lo:up + 1] & mask, b[lo:up + 1] & mask)
        assert np.array_equal(np.sort(a[lo:up + 1]), np.sort(b[lo:up + 1]))
        assert cb.tolist() == ca.tolist(), pos


# --------------------------------------------------------------------------
# distributions and edge cases (reference tests/test_variants.py)
# --------------------------------------------------------------------------

DISTS = {
    "low16_u64": lambda n: cases.config3("low16", n),
    "zipf_u64": lambda n: cases.config3("zipf", n),
    "uniform_u64": lambda n: cases.config3("uniform", n),
    "sorted_u32": lambda n: np.arange(n, dtype=np.uint32) * np.uint32(7),
    "reverse_u32": lambda n: (np.arange(n, dtype=np.uint32) * np.uint32(7))[::-1].copy(),
    "all_equal_u32": lambda n: np.full(n, 0xDEADBEEF, np.uint32),
    "two_values_u32": lambda n: (np.random.default_rng(1).integers(0, 2, n) * 0xFFFFFFFF).astype(np.uint32),
    "few_u64": lambda n: np.random.default_rng(2).integers(0, 5, n).astype(np.uint64) << np.uint64(40),
    "dup_heavy_u32": lambda n: np.random.default_rng(4).integers(0, 300, n).astype(np.uint32) * np.uint32(65537),
    "dense16_u32": lambda n: np.random.default_rng(5).integers(0, 1 << 16, n).astype(np.uint32),
    # dense local-sort tasks with second/third/fourth+ copies (B2, B3, overflow list)
    "dense_dups_u32": lambda n: _top_low(6, n, 1 << 10, 1 << 12),
    "dense_dups_sparse_u32": lambda n: _top_low(7, n, 1 << 10, 1 << 13),
    # ~4096-key dense tasks over 2^14 values: a few dozen third copies each (the small variant's
    # overflow list, below its hand-over threshold)
    "dense_list_u32": lambda n: _top_low(13, n, 1 << 10, 1 << 14),
    # ~6500-key big dense tasks with 4 distinct low halves each: the big variant's overflow list runs
    # over and every task is handed to the general local sort (a bucket list sized for > 8192-key
    # buckets must not receive them: found by tools/fuzz_gpu.py)
    "big_dense_handover_u32": lambda n: _top_low(14, n, 640, 4),
    # ~16K-key tasks for the big dense variant, with a few repeats
    "big_dense_u32": lambda n: _top_low(8, n, 1 << 8, 1 << 16),
    # local bin sort: equal keys ranked inside a bin (each value 2 / 3 times) and
    # the comparison-budget fallback to LSD (each value 41 times)
    "dup2_u64": lambda n: _repeated(9, n, 2),
    "dup3_u32": lambda n: _repeated(12, n, 3).astype(np.uint32),
    "dup41_u64": lambda n: _repeated(10, n, 41),
    # sorted runs in random order (hist16 warp-aggregated bins for some warps only)
    "sorted_runs_u32": lambda n: _sorted_runs(11, n, 1000),
}


def _repeated(seed, n, k):
    """u64 keys: random values, each repeated k times, shuffled."""
    r = np.random.default_rng(seed)
    v = r.integers(0, 1 << 63, (n + k - 1) // k, dtype=np.uint64) * np.uint64(2)
    x = np.repeat(v, k)[:n]
    r.shuffle(x)
    return x


def _sorted_runs(seed, n, run):
    r = np.random.default_rng(seed)
    x = np.sort(r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32))
    blocks = [x[i:i + run] for i in range(0, n, run)]
    order = r.permutation(len(blocks))
    return np.concatenate([blocks[i] for i in order])


def _top_low(seed, n, ntop, nlow):
    """u32 keys: top 16 bits from `ntop` values, low 16 bits from [0, nlow)."""
    r = np.random.default_rng(seed)
    top = (r.integers(0, ntop, n).astype(np.uint32) * np.uint32(40503)) & np.uint32(0xFFFF)
    return (top << np.uint32(16)) | r.integers(0, nlow, n).astype(np.uint32)


@pytest.mark.parametrize("name", sorted(DISTS))
def test_distributions(cuda, name):
    x = DISTS[name](1 << 22)
    got = x.copy()
    bs.sort(got, UnsignedCodec(x.dtype.itemsize * 8), with_metrics=False)
    assert np.array_equal(got, np.sort(x))


def test_edge_sizes(cuda):
    for n in (0, 1, 2, 7, 8192, 8193, 6144, 6145):
        x = np.random.default_rng(n).integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
        got = x.copy()
        bs.sort(got, UnsignedCodec(32))
        assert np.array_equal(got, np.sort(x))


def test_sequence_kinds(cuda):
    import torch

    rng = np.random.default_rng(11)
    base = rng.integers(0, 2 ** 32, 10000, dtype=np.uint64).astype(np.uint32)
    # strided numpy view is sorted in place through the view
    y = np.repeat(base, 2)
    bs.sort(y[::2], UnsignedCodec(32))
    assert np.array_equal(y[::2], np.sort(base)) and np.array_equal(y[1::2], base)
    # python list of ints
    lst = [int(v) for v in base[:500]]
    bs.sort(lst, UnsignedCodec(32))
    assert lst == sorted(int(v) for v in base[:500])
    # CUDA tensor sorted in place on its device
    t = torch.from_numpy(base.view(np.int32)).cuda()
    bs.sort(t, UnsignedCodec(32))
    assert np.array_equal(t.cpu().numpy().view(np.uint32), np.sort(base))
    # CPU tensor: copied in and back
    c = torch.from_numpy(base.view(np.int32).copy())
    bs.sort(c, UnsignedCodec(32))
    assert np.array_equal(c.numpy().view(np.uint32), np.sort(base))
    # read-only arrays are rejected instead of crashing like the reference
    ro = base.copy()
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        bs.sort(ro, UnsignedCodec(32))


def test_signed_and_float_codecs(cuda):
    rng = np.random.default_rng(12)
    x = rng.integers(-2 ** 31, 2 ** 31, 200000).astype(np.int32)
    g = x.copy()
    bs.sort(g, SignedCodec(32))
    assert np.array_equal(g, np.sort(x))
    s8 = [5, -3, 127, -128, 0, -1]
    bs.sort(s8, SignedCodec(8))
    assert s8 == sorted(s8)
    f = rng.standard_normal(100000)
    f[:8] = [np.inf, -np.inf, 0.0, -0.0, np.nan, -np.nan, 1e-300, -1e-300]
    g = f.copy()
    bs.sort(g, Float64Codec())
    u = f.view(np.uint64)
    enc = np.where(u >> np.uint64(63), ~u, u | np.uint64(1 << 63))
    assert np.array_equal(g.view(np.uint64), u[np.argsort(enc, kind="stable")])
    # reference tests/test_keys.py:168-172 golden order
    h = [1.5, -0.0, np.inf, -3.25, 0.0, -np.inf]
    bs.sort(h, Float64Codec())
    assert [repr(v) for v in h] == [repr(v) for v in [-np.inf, -3.25, -0.0, 0.0, 1.5, np.inf]]


# --------------------------------------------------------------------------
# key-value (cfg4 shape) and variants
# --------------------------------------------------------------------------

def test_kv_stable_pairs(cuda):
    k, p = cases.config4(1 << 22)
    kk, pp = k.copy(), p.copy()
    bs.sort(kk, UnsignedCodec(32), values=pp, with_metrics=False)
    order = np.argsort(k, kind="stable")
    assert np.array_equal(kk, k[order]) and np.array_equal(pp, p[order])
    assert np.array_equal(k[pp], kk)  # every payload stays with its key


def test_kv_equals_packed_word_sort(cuda, oracle_lib):
    # stable KV order == reference sort of (key << 32 | index)
    k, p = cases.config4(1 << 18)
    packed = (k.astype(np.uint64) << np.uint64(32)) | p.astype(np.uint64)
    oracle_lib.sort(packed, 64)
    kk, pp = k.copy(), p.copy()
    bs.sort(kk, UnsignedCodec(32), values=pp, with_metrics=False)
    assert np.array_equal(kk, (packed >> np.uint64(32)).astype(np.uint32))
    assert np.array_equal(pp, (packed & np.uint64(0xFFFFFFFF)).astype(np.uint32))


def test_kv_u64_keys_u64_values(cuda):
    rng = np.random.default_rng(13)
    k = rng.integers(0, 1000, 300000).astype(np.uint64) << np.uint64(33)
    v = rng.integers(0, 2 ** 64, k.size, dtype=np.uint64)
    kk, vv = k.copy(), v.copy()
    bs.sort(kk, UnsignedCodec(64), values=vv, with_metrics=False)
    order = np.argsort(k, kind="stable")
    assert np.array_equal(kk, k[order]) and np.array_equal(vv, v[order])


@pytest.mark.parametrize("kdt,vdt", [(np.uint32, np.uint64), (np.uint64, np.uint32), (np.uint32, np.uint32)])
def test_kv_mixed_widths_stable(cuda, kdt, vdt):
    # several scatter levels (tiles of the stable scatter + tile scan) and ties
    rng = np.random.default_rng(14)
    n = (1 << 22) + 12345
    bits = 8 * np.dtype(kdt).itemsize
    k = (rng.integers(0, 1 << 20, n, dtype=np.uint64) << np.uint64(bits - 20)).astype(kdt)
    v = rng.integers(0, np.iinfo(vdt).max, n, dtype=np.uint64).astype(vdt)
    kk, vv = k.copy(), v.copy()
    bs.sort(kk, UnsignedCodec(bits), values=vv, with_metrics=False)
    order = np.argsort(k, kind="stable")
    assert np.array_equal(kk, k[order]) and np.array_equal(vv, v[order])


def test_variants_same_output(cuda):
    rng = np.random.default_rng(40)
    base = rng.integers(0, 2 ** 32, 200000, dtype=np.uint64).astype(np.uint32)
    want = np.sort(base)
    for fn in (lambda s: bs.sort_iterative(s, UnsignedCodec(32)),
               lambda s: bs.sort_optimized(s, UnsignedCodec(32)),
               lambda s: bs.sort_parallel(s, UnsignedCodec(32), 8)):
        w = base.copy()
        fn(w)
        assert np.array_equal(w, want)


def test_range_sorted_words(cuda):
    assert kernels.range_sorted_words(np.array([1, 2, 2, 9], dtype=np.uint32), 0, 3)
    assert not kernels.range_sorted_words(np.array([1, 3, 2], dtype=np.uint32), 0, 2)
    assert kernels.range_sorted_words(np.array([3, 1, 2], dtype=np.uint32), 1, 2)


# --------------------------------------------------------------------------
# multi-GPU device steps on one GPU (split + sample); R=1 dist path
# --------------------------------------------------------------------------

def test_split_by_splitters_device_step(cuda):
    import torch

    from paper_0811_3448_b200.dist import CudaOps

    rng = np.random.default_rng(14)
    k = rng.integers(0, 2 ** 32, 100000, dtype=np.uint64).astype(np.uint32)
    k[:20000] = 777777
    v = np.arange(k.size, dtype=np.uint32)
    ops = CudaOps(32)
    kt = torch.from_numpy(k.view(np.int32)).cuda()
    vt = torch.from_numpy(v.view(np.int32)).cuda()
    spl = np.array([777777, 2 ** 31, 3 * 2 ** 30], dtype=np.uint32)
    ok, ov, cnt = ops.split(kt, vt, torch.from_numpy(spl.view(np.int32)).cuda(), 4)
    cls = 2 * (spl[None, :] < k[:, None]).sum(1) + (spl[None, :] == k[:, None]).any(1)
    order = np.argsort(cls, kind="stable")
    assert cnt.cpu().numpy().tolist() == np.bincount(cls, minlength=7).tolist()
    assert np.array_equal(ok.cpu().numpy().view(np.uint32), k[order])
    assert np.array_equal(ov.cpu().numpy().view(np.uint32), v[order])
    smp = ops.sample(kt, 64).cpu().numpy().view(np.uint32)
    assert np.array_equal(smp, k[[(2 * i + 1) * k.size // 128 for i in range(64)]])


def test_dist_sort_single_rank(cuda):
    import torch

    from paper_0811_3448_b200.dist import dist_sort

    x = cases.mt_words(9, 1 << 20)
    t = torch.from_numpy(x.view(np.int32)).cuda()
    r = dist_sort(t, width=32)
    assert np.array_equal(r.keys.cpu().numpy().view(np.uint32), np.sort(x))


# --------------------------------------------------------------------------
# full BASELINE.json sizes vs the reference's own outputs (golden hashes)
# --------------------------------------------------------------------------

def _sort_dev(x, values=None):
    import torch

    t = torch.from_numpy(x.view(np.int32 if x.itemsize == 4 else np.int64)).cuda()
    v = None if values is None else torch.from_numpy(values.view(np.int32)).cuda()
    device.sort_words_device(t, v, width=x.itemsize * 8)
    out = t.cpu().numpy().view(x.dtype)
    device.workspaces.clear()
    return out, (None if v is None else v.cpu().numpy().view(values.dtype))


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg2", "cfg3_uniform", "cfg3_zipf", "cfg3_low16", "cfg4_packed",
                                  "cfg5", "cfg5_sorted", "cfg5_reverse"])
def test_full_size_configs_match_reference(cuda, golden, name):
    g = golden.get("big", {}).get(name)
    if g is None:
        pytest.skip("golden.json was generated without --big")
    if name == "cfg2":
        x = cases.config2()
    elif name.startswith("cfg3"):
        x = cases.config3(name.split("_")[1])
    elif name == "cfg4_packed":
        k, p = cases.config4()
        out_k, out_p = _sort_dev(k, p)
        assert sha(out_k) == g["keys_sha"] and sha(out_p) == g["payload_sha"]
        return
    else:
        x = cases.config5("uniform")
        if name == "cfg5_sorted":
            x.sort()
        elif name == "cfg5_reverse":
            x = np.sort(x)[::-1].copy()
    assert sha(x) == g["input_sha"]
    out, _ = _sort_dev(x)
    assert sha(out) == g["output_sha"]


# --------------------------------------------------------------------------
# level-0 digit-pair histogram (hist16): bins past 32767 spill to the global
# counts; constant second digits requeue with a real histogram pass
# --------------------------------------------------------------------------

def _heavy_prefix(n, seed):
    """u32 keys, 7/8 of them under one 16-bit prefix (every CTA's bin spills)."""
    r = np.random.default_rng(seed)
    x = r.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    heavy = r.random(n) < 0.875
    x[heavy] = np.uint32(0xBEEF0000) | (x[heavy] & np.uint32(0xFFFF))
    return x


@pytest.mark.parametrize("kv", [False, True])
def test_hist16_spills_exact(cuda, kv):
    x = _heavy_prefix(1 << 24, 21)
    if kv:
        p = np.arange(x.size, dtype=np.uint32)
        kk, pp = x.copy(), p.copy()
        bs.sort(kk, UnsignedCodec(32), values=pp, with_metrics=False)
        order = np.argsort(x, kind="stable")
        assert np.array_equal(kk, x[order]) and np.array_equal(pp, p[order])
    else:
        got = x.copy()
        bs.sort(got, UnsignedCodec(32), with_metrics=False)
        assert np.array_equal(got, np.sort(x))


@pytest.mark.parametrize("head", [0, 1, 3])
def test_sorted_input_unaligned_views(cuda, head):
    # already-sorted / reverse-sorted device views starting off a 16-byte boundary:
    # hist16's warp-uniform bin adds must count ragged head and tail granules exactly
    import torch

    from paper_0811_3448_b200 import device

    n = (1 << 22) + 5
    base = np.sort(np.random.default_rng(23).integers(0, 1 << 32, n + head, dtype=np.uint64).astype(np.uint32))
    for x in (base, base[::-1].copy()):
        t = torch.from_numpy(x.view(np.int32)).cuda()
        v = t[head:]
        device.sort_words_device(v, width=32)
        got = v.cpu().numpy().view(np.uint32)
        assert np.array_equal(got, np.sort(x[head:]))
        assert np.array_equal(t[:head].cpu().numpy().view(np.uint32), x[:head])


def test_hist16_constant_second_digit(cuda):
    # every root child has a constant second digit (one occupied hist16 bin per row)
    r = np.random.default_rng(22)
    top = r.integers(0, 256, 1 << 23).astype(np.uint32)
    x = (top << np.uint32(24)) | ((top * np.uint32(37)) & np.uint32(0xFF)) << np.uint32(16) | \
        r.integers(0, 1 << 16, top.size).astype(np.uint32)
    got = x.copy()
    bs.sort(got, UnsignedCodec(32), with_metrics=False)
    assert np.array_equal(got, np.sort(x))


# --------------------------------------------------------------------------
# whole-input counting (gen16): every varying bit inside the hist16 digit pair
# --------------------------------------------------------------------------

@pytest.mark.parametrize("case", ["u32_low16", "u32_mid16", "u32_top16", "u32_skew", "u64_mid16", "u64_low9",
                                  "i32_low16", "f64_span", "u32_straddle"])
def test_whole_input_counting(cuda, case):
    rng = np.random.default_rng(hash(case) % 2 ** 32)
    n = (1 << 22) + 12345
    if case == "u32_low16":
        x = (rng.integers(0, 1 << 16, n, dtype=np.uint64) | 0xABCD0000).astype(np.uint32)
    elif case == "u32_mid16":
        x = ((rng.integers(0, 1 << 16, n, dtype=np.uint64) << 8) | 0x9E000077).astype(np.uint32)
    elif case == "u32_top16":
        x = ((rng.integers(0, 1 << 16, n, dtype=np.uint64) << 16) | 0x1234).astype(np.uint32)
    elif case == "u32_skew":
        x = rng.integers(0, 1 << 16, n, dtype=np.uint64).astype(np.uint32)
        x[rng.random(n) < 0.9] = 77
    elif case == "u64_mid16":
        x = (rng.integers(0, 1 << 16, n, dtype=np.uint64) << np.uint64(24)) | np.uint64(0x5555000000FFFFFF)
    elif case == "u64_low9":
        x = rng.integers(0, 1 << 9, n, dtype=np.uint64) | np.uint64(0xFEDCBA9876540000)
    elif case == "i32_low16":
        x = (rng.integers(-(1 << 15), 1 << 15, n)).astype(np.int32)
    elif case == "f64_span":
        x = np.frombuffer((rng.integers(0, 1 << 16, n, dtype=np.uint64) << np.uint64(30) |
                           np.uint64(0x4010000000000000)).tobytes(), dtype=np.float64).copy()
    else:  # varying bits straddle the pair: the ordinary MSD path
        x = ((rng.integers(0, 1 << 18, n, dtype=np.uint64) << 7)).astype(np.uint32)
    codec = {np.dtype(np.uint32): UnsignedCodec(32), np.dtype(np.uint64): UnsignedCodec(64),
             np.dtype(np.int32): SignedCodec(32), np.dtype(np.float64): Float64Codec()}[x.dtype]
    a = x.copy()
    m = bs.sort(a, codec)
    want = np.sort(x) if x.dtype.kind != "f" else x[np.argsort(x, kind="stable")]
    assert np.array_equal(a.view(np.uint8), want.view(np.uint8)), case
    assert m.bit_extractions > 0
