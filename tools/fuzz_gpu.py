"""Randomised differential test of the CUDA sort against numpy (run on a GPU box).

    python tools/fuzz_gpu.py [--seconds 300] [--seed 0] [--max-log2 24] [--dist]

Random sizes, key types (u32 / u64 / i32 / f64), distributions (uniform, few
distinct values, sorted / reverse runs, top-bits x low-bits products that make
dense tasks of every size, low-entropy words), unaligned views, and key-value
sorts (stable order).  With --dist: the multi-GPU device steps with 2..8
emulated ranks on the one GPU (sample, class count, fused exchange into R
receive buffers, local sort; shards of random and empty sizes), keys only and
key-value (global stable order).  Prints one line per failure and a summary;
exit 1 on any mismatch.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def gen(r: np.random.Generator, n: int, bits: int) -> np.ndarray:
    dt = np.uint32 if bits == 32 else np.uint64
    kind = int(r.integers(0, 8))
    if kind == 0:
        x = r.integers(0, 2 ** bits, n, dtype=np.uint64)
    elif kind == 1:  # few distinct values
        vals = r.integers(0, 2 ** bits, int(r.integers(1, 2000)), dtype=np.uint64)
        x = vals[r.integers(0, vals.size, n)]
    elif kind == 2:  # sorted runs
        x = np.sort(r.integers(0, 2 ** bits, n, dtype=np.uint64))
        if r.integers(0, 2):
            x = x[::-1]
    elif kind == 3:  # top x low product: dense tasks of many sizes and multiplicities
        ntop = 1 << int(r.integers(0, 17))
        nlow = 1 << int(r.integers(1, 17))
        top = r.integers(0, ntop, n, dtype=np.uint64) * np.uint64(40503) % np.uint64(1 << 16)
        x = (top << np.uint64(bits - 16)) | r.integers(0, nlow, n, dtype=np.uint64) << np.uint64(int(r.integers(0, bits - 31)))
    elif kind == 4:  # low-entropy: random bits under a random mask
        mask = r.integers(0, 2 ** bits, dtype=np.uint64)
        x = r.integers(0, 2 ** bits, n, dtype=np.uint64) & mask
    elif kind == 5:  # zipf-like
        vals = r.integers(0, 2 ** bits, 1 << 12, dtype=np.uint64)
        x = vals[np.minimum(r.zipf(1.2, n) - 1, vals.size - 1)]
    elif kind == 6:  # only the low 16 (or fewer) bits
        x = r.integers(0, 1 << int(r.integers(1, 17)), n, dtype=np.uint64) << np.uint64(int(r.integers(0, bits - 15)))
    else:  # nearly sorted
        x = np.sort(r.integers(0, 2 ** bits, n, dtype=np.uint64))
        k = max(1, n // 100)
        i = r.integers(0, n, k)
        x[i] = r.integers(0, 2 ** bits, k, dtype=np.uint64)
    return (x & np.uint64(2 ** bits - 1)).astype(dt)


def emulated_ranks(shards, vals, R):
    """The per-rank device steps of dist_sort with a destination table on this GPU (tests/test_gpu_dist.py)."""
    import types

    import torch

    from paper_0811_3448_b200.dist import CudaOps, choose_splitters, exchange_plan

    kb = shards[0].dtype.itemsize
    sdt = {4: torch.int32, 8: torch.int64}[kb]
    ndt = {4: np.int32, 8: np.int64}[kb]
    udt = {4: np.uint32, 8: np.uint64}[kb]
    ops = CudaOps(kb * 8, 0)
    keys = [torch.from_numpy(s.view(ndt)).cuda() for s in shards]
    vt = [torch.from_numpy(v.view(np.int32)).cuda() for v in vals] if vals is not None else None
    smp = torch.cat([ops.sample(k, 4096 if k.numel() else 0) for k in keys])
    ss = ops.sort_samples(smp).cpu().numpy().view(udt)
    spl = torch.from_numpy(choose_splitters(ss, R).view(ndt)).cuda()
    # one CudaOps per source rank: the exchange reads the tile offsets its own class count left in
    # that rank's workspace
    per = [CudaOps(kb * 8, 0) for _ in range(R)]
    cc = np.array([per[r].split_count(keys[r], spl, R).cpu().numpy() for r in range(R)], dtype=np.int64)
    _, _, rcounts = exchange_plan(cc, R, 0)
    recv_k = [torch.empty(max(1, int(c)), dtype=sdt, device="cuda") for c in rcounts]
    recv_v = [torch.empty(max(1, int(c)), dtype=torch.int32, device="cuda") for c in rcounts] if vals else None
    bufs = types.SimpleNamespace(
        key_table=torch.tensor([t.data_ptr() for t in recv_k], dtype=torch.int64, device="cuda"),
        val_table=torch.tensor([t.data_ptr() for t in recv_v], dtype=torch.int64, device="cuda") if vals else None)
    for r in range(R):
        B, delta, _ = exchange_plan(cc, R, r)
        if keys[r].numel():
            per[r].exchange(keys[r], vt[r] if vt else None, spl, R, delta, B, bufs)
    outk, outv = [], []
    for d in range(R):
        b = types.SimpleNamespace(device=recv_k[d].device, local_keys=recv_k[d].data_ptr(),
                                  local_vals=recv_v[d].data_ptr() if vals else None)
        k, v = ops.sort_from(b, int(rcounts[d]), sdt, torch.int32 if vals else None)
        outk.append(k.cpu().numpy().view(udt))
        if vals:
            outv.append(v.cpu().numpy().view(np.uint32))
    return np.concatenate(outk), (np.concatenate(outv) if vals else None)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-log2", type=int, default=24)
    ap.add_argument("--dist", action="store_true", help="fuzz the multi-GPU device steps with emulated ranks")
    a = ap.parse_args(argv)
    import torch

    import paper_0811_3448_b200 as bs
    from paper_0811_3448_b200 import Float64Codec, SignedCodec, UnsignedCodec

    r = np.random.default_rng(a.seed)
    t0 = time.time()
    runs = fails = 0
    while time.time() - t0 < a.seconds:
        n = int(2 ** r.uniform(0, a.max_log2)) + int(r.integers(0, 3))
        bits = 32 if r.integers(0, 2) else 64
        x = gen(r, n, bits)
        mode = int(r.integers(0, 6))
        head = int(r.integers(0, 4))
        what = f"n={n} bits={bits} mode={mode} head={head} seed={a.seed} run={runs}"
        try:
            if a.dist:
                R = int(r.integers(2, 9))
                cuts = np.sort(r.integers(0, n + 1, R - 1)) if r.integers(0, 3) else \
                    np.array([(i + 1) * n // R for i in range(R - 1)])
                shards = [s_.copy() for s_ in np.split(x, cuts)]
                kv = bool(r.integers(0, 2))
                vals = [np.arange(s_.size, dtype=np.uint32) | np.uint32(i << 28) for i, s_ in enumerate(shards)] if kv else None
                what += f" R={R} kv={kv} sizes={[s_.size for s_ in shards]}"
                gk, gv = emulated_ranks(shards, vals, R)
                allk = np.concatenate(shards)
                if kv:
                    allv = np.concatenate(vals)
                    order = np.argsort(allk, kind="stable")
                    ok = np.array_equal(gk, allk[order]) and np.array_equal(gv, allv[order])
                else:
                    ok = np.array_equal(gk, np.sort(allk))
            elif mode <= 2:  # keys only, device tensor view (possibly unaligned start)
                buf = torch.empty(n + head, dtype=torch.int32 if bits == 32 else torch.int64, device="cuda")
                view = buf[head:]
                view.copy_(torch.from_numpy(x.view(np.int32 if bits == 32 else np.int64)))
                bs.sort(view, UnsignedCodec(bits), with_metrics=False)
                got = view.cpu().numpy().view(x.dtype)
                ok = np.array_equal(got, np.sort(x))
            elif mode == 3 and bits == 32:  # signed
                y = x.view(np.int32).copy()
                bs.sort(y, SignedCodec(32), with_metrics=False)
                ok = np.array_equal(y, np.sort(x.view(np.int32)))
            elif mode == 3:  # float64 total order (no NaN payload subtleties: compare bit patterns of finite values)
                f = x.view(np.float64).copy()
                f = f[np.isfinite(f)]
                w = f.copy()
                bs.sort(w, Float64Codec(), with_metrics=False)
                ok = np.array_equal(w, np.sort(f)) if f.size else True
            else:  # key-value, stable
                v = np.arange(n, dtype=np.uint32)
                k = torch.from_numpy(x.view(np.int32 if bits == 32 else np.int64)).cuda()
                vv = torch.from_numpy(v.view(np.int32)).cuda()
                bs.sort(k, UnsignedCodec(bits), values=vv, with_metrics=False)
                order = np.argsort(x, kind="stable")
                ok = np.array_equal(k.cpu().numpy().view(x.dtype), x[order]) and \
                    np.array_equal(vv.cpu().numpy().view(np.uint32), v[order])
        except Exception as e:  # noqa: BLE001
            ok = False
            what += f" EXC {e!r}"
        runs += 1
        if not ok:
            fails += 1
            print("FAIL", what, flush=True)
            if "EXC" in what and "Accelerator" in what:
                break  # the CUDA context is gone: nothing after this is meaningful
    print(f"fuzz: {runs} runs, {fails} failures, {time.time() - t0:.0f} s", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
