"""Small sorts that exercise every kernel family.  Run them against the
bounds-checked build (tests/test_gpu_debug_checks.py does):

    BS_LIBRARY=debug python tools/sanitize_cases.py

(compute-sanitizer is closed on this GPU pool; the checked build replaces it.)

keys-only u32 (hist16, scatter_ws, dense, local), u64 (bin/LSD local sort),
key-value (stable scatter with tile_scan look-back), signed/float codecs,
the exact reference-order engine, the partition pass, and the multi-GPU
device steps (sample, class count, fused exchange into R=3 receive buffers,
sort_from).  Every result is checked against numpy.
"""
import os
import sys
import types

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_0811_3448_b200 import _lib, device  # noqa: E402
from paper_0811_3448_b200.dist import CudaOps, exchange_plan  # noqa: E402


def words(dt, n, seed, hi=None):
    r = np.random.default_rng(seed)
    bits = np.dtype(dt).itemsize * 8
    return r.integers(0, hi or 2 ** bits, n, dtype=np.uint64).astype(dt)


def dev(x):
    return torch.from_numpy(x.view({4: np.int32, 8: np.int64}[x.itemsize]).copy()).cuda()


def check(d, want, what):
    got = d.cpu().numpy().view(want.dtype)
    assert np.array_equal(got, want), what
    print("ok", what, flush=True)


if os.environ.get("BS_LIBRARY") == "debug":
    assert _lib.lib().bs_debug_checks() == 1, "BS_LIBRARY=debug did not load the checked build"
    print("checked build loaded", flush=True)
n = int(os.environ.get("BS_SAN_N", 1 << 18))
x = words(np.uint32, n, 1)
d = dev(x)
device.sort_words_device(d, width=32)
check(d, np.sort(x), "u32 keys (hist16/scatter/dense)")
big = words(np.uint32, 1 << 22, 11)
d = dev(big)
device.sort_words_device(d, width=32)
check(d, np.sort(big), "u32 2^22 keys (two scatter levels)")
# dense tasks of ~4096 keys with second / third copies and overflow-list entries, and ~16K-key big ones
for ntop, nlow, what in ((1 << 10, 1 << 14, "small dense tasks, listed copies"), (1 << 10, 1 << 12, "small dense tasks, hand-over"),
                         (1 << 8, 1 << 16, "big dense tasks")):
    r = np.random.default_rng(ntop + nlow)
    top = (r.integers(0, ntop, 1 << 22).astype(np.uint32) * np.uint32(40503)) & np.uint32(0xFFFF)
    dd = (top << np.uint32(16)) | r.integers(0, nlow, 1 << 22).astype(np.uint32)
    d = dev(dd)
    device.sort_words_device(d, width=32)
    check(d, np.sort(dd), "u32 " + what)
y = words(np.uint32, n, 2, hi=300) * np.uint32(65537)
d = dev(y)
device.sort_words_device(d, width=32)
check(d, np.sort(y), "u32 heavy ties (local)")
z = words(np.uint64, n // 2, 3)
d = dev(z)
device.sort_words_device(d, width=64)
check(d, np.sort(z), "u64 keys")
k = words(np.uint32, n, 4, hi=1024)
v = np.arange(n, dtype=np.uint32)
dk, dv = dev(k), dev(v)
device.sort_words_device(dk, dv, width=32)
o = np.argsort(k, kind="stable")
check(dk, k[o], "kv keys (stable scatter + look-back)")
check(dv, v[o], "kv values")
s = words(np.uint32, n // 4, 5).view(np.int32)
d = torch.from_numpy(s.copy()).cuda()
device.sort_words_device(d, width=32, key_kind=_lib.BS_KEY_SIGNED)
check(d, np.sort(s), "signed codec")
f = np.random.default_rng(6).standard_normal(n // 4)
d = torch.from_numpy(f.view(np.int64).copy()).cuda()
device.sort_words_device(d, width=64, key_kind=_lib.BS_KEY_FLOAT)
assert np.array_equal(d.cpu().numpy().view(np.float64), np.sort(f))
print("ok float codec", flush=True)
e = words(np.uint64, 20000, 7)
d = dev(e)
c = torch.zeros(4, dtype=torch.int64, device="cuda")
device.exact_sort_device(d, width=32, mode=_lib.EX_REC, passthrough_loop=True, check_after=2, counters=c)
# the reference's sortedness scan compares whole words, so with width < 64 a
# range may stop early unsorted in its low bits: check the multiset only
assert np.array_equal(np.sort(d.cpu().numpy().view(np.uint64)), np.sort(e))
print("ok exact engine", flush=True)
p = words(np.uint32, 50000, 8)
d = dev(p)
device.partition_device(d, width=32, pos=3)
print("ok partition", flush=True)
# multi-GPU device steps with three emulated ranks
R = 3
shards = [words(np.uint32, n // 3 + 11 * r, 20 + r) for r in range(R)]
keys = [dev(sh) for sh in shards]
ops = CudaOps(32)
smp = torch.cat([ops.sample(kk, 1024) for kk in keys])
ss = ops.sort_samples(smp)
spl = ss[torch.arange(1, R, device="cuda") * 1024].contiguous()
per = [CudaOps(32) for _ in range(R)]
cc = np.array([per[r].split_count(keys[r], spl, R).cpu().numpy() for r in range(R)], dtype=np.int64)
_, _, rc = exchange_plan(cc, R, 0)
recv = [torch.empty(max(1, int(q)), dtype=torch.int32, device="cuda") for q in rc]
bufs = types.SimpleNamespace(key_table=torch.tensor([t.data_ptr() for t in recv], dtype=torch.int64, device="cuda"),
                             val_table=None)
for r in range(R):
    B, delta, _ = exchange_plan(cc, R, r)
    per[r].exchange(keys[r], None, spl, R, delta, B, bufs)
out = []
for dd in range(R):
    b = types.SimpleNamespace(device=recv[dd].device, local_keys=recv[dd].data_ptr(), local_vals=None)
    kk, _ = ops.sort_from(b, int(rc[dd]), torch.int32, None)
    out.append(kk.cpu().numpy().view(np.uint32))
assert np.array_equal(np.concatenate(out), np.sort(np.concatenate(shards)))
print("ok dist device steps", flush=True)
torch.cuda.synchronize()
print("ALL OK")
