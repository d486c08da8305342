"""Time the multi-GPU device steps on ONE GPU with emulated ranks.

R shards of `--keys-per-rank` uint32 keys (MT19937 streams) live on cuda:0;
every "rank" runs its real device steps -- bs_split_count (class histogram +
scan) and bs_split_exchange (fused partition + stores into the destination
ranks' receive buffers) -- with a destination table that points at R receive
buffers on the same device (on an NVSwitch node these are peer mappings), then
bs_sort_from on each receive buffer.  Prints one JSON line with per-step
CUDA-event times and the achieved bytes/s of the count and exchange kernels.

    python tools/exchange_bench.py [--ranks 8] [--keys-per-rank 33554432]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--keys-per-rank", type=int, default=1 << 25)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args(argv)
    import torch

    from paper_0811_3448_b200.cases import mt_words
    from paper_0811_3448_b200.dist import CudaOps, exchange_plan

    R, n = a.ranks, a.keys_per_rank
    keys = [torch.from_numpy(mt_words(1 + r, n).view(np.int32)).cuda() for r in range(R)]
    ops = [CudaOps(32) for _ in range(R)]
    smp = torch.cat([ops[0].sample(k, 4096) for k in keys])
    ss = ops[0].sort_samples(smp)
    spl = ss[torch.arange(1, R, device="cuda") * 4096].contiguous()
    cc = np.array([ops[r].split_count(keys[r], spl, R).cpu().numpy() for r in range(R)], dtype=np.int64)
    _, _, rc = exchange_plan(cc, R, 0)
    recv = [torch.empty(int(c) + 1, dtype=torch.int32, device="cuda") for c in rc]
    bufs = types.SimpleNamespace(key_table=torch.tensor([t.data_ptr() for t in recv], dtype=torch.int64,
                                                        device="cuda"), val_table=None)
    plans = [exchange_plan(cc, R, r) for r in range(R)]

    def ev():
        return torch.cuda.Event(enable_timing=True)

    t_count, t_exch, t_sort = [], [], []
    for rep in range(a.reps + 1):
        e = [ev() for _ in range(4)]
        e[0].record()
        for r in range(R):
            ops[r].split_count(keys[r], spl, R)
        e[1].record()
        for r in range(R):
            B, delta, _ = plans[r]
            ops[r].exchange(keys[r], None, spl, R, delta, B, bufs)
        e[2].record()
        outs = []
        for d in range(R):
            b = types.SimpleNamespace(device=recv[d].device, local_keys=recv[d].data_ptr(), local_vals=None)
            outs.append(ops[0].sort_from(b, int(rc[d]), torch.int32, None)[0])
        e[3].record()
        torch.cuda.synchronize()
        if rep:
            t_count.append(e[0].elapsed_time(e[1]))
            t_exch.append(e[1].elapsed_time(e[2]))
            t_sort.append(e[2].elapsed_time(e[3]))
    allk = np.concatenate([k.cpu().numpy().view(np.uint32) for k in keys])
    got = np.concatenate([o.cpu().numpy().view(np.uint32) for o in outs])
    ok = bool(np.array_equal(got, np.sort(allk)))
    N = R * n
    mc, me, ms = (float(np.median(t)) for t in (t_count, t_exch, t_sort))
    print(json.dumps({
        "ranks_emulated": R, "keys_per_rank": n, "correct": ok,
        "count_ms_all_ranks": mc, "count_GBps": 4 * N / (mc / 1e3) / 1e9,
        "exchange_ms_all_ranks": me, "exchange_GBps_read_plus_write": 8 * N / (me / 1e3) / 1e9,
        "local_sort_ms_all_ranks": ms,
        "note": "all ranks' steps serialised on one GPU; receive buffers local (peer stores on a real node)"}))
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
