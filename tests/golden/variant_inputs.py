"""Seeded inputs shared by make_golden_variants.py (run against the reference)
and the tests (run against the GPU): both regenerate the same words and the
golden file pins each one by its sha256."""

import numpy as np

KINDS = ("random", "sorted", "ties", "nearly", "lowvar")


def words(kind: str, bits: int, width: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    dt = np.uint32 if bits == 32 else np.uint64
    full = rng.integers(0, 2 ** bits, n, dtype=np.uint64)
    above = np.uint64(0) if width >= 64 else (full >> np.uint64(width)) << np.uint64(width)
    above = above & np.uint64((1 << bits) - 1)
    if kind == "random":
        x = full
    elif kind == "sorted":
        x = np.sort(full)
    elif kind == "ties":  # 7 distinct keys, random bits above the key
        x = above | rng.integers(0, 7, n, dtype=np.uint64)
    elif kind == "nearly":  # sorted with a few swapped pairs
        x = np.sort(full)
        for _ in range(max(1, n // 100)):
            i, j = rng.integers(0, n, 2)
            x[i], x[j] = x[j], x[i]
    elif kind == "lowvar":  # one constant key prefix, 6 varying low bits: long pass-through streaks
        base = np.uint64(int(rng.integers(0, 2 ** min(width, 63))) & ~0x3F & ((1 << width) - 1))
        x = above | base | (full & np.uint64(0x3F))
        if n > 8:
            x[: n // 2] = np.sort(x[: n // 2])
    else:
        raise ValueError(kind)
    return x.astype(dt)
