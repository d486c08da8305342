"""Seeded synthetic inputs (drop-in for the generator half of ``binarsort.oracle``).

* :class:`MT19937` -- the classic 32-bit Mersenne Twister with the standard
  1812433253 initialiser (reference ``oracle.py:34-108``).  numpy's
  ``MT19937._legacy_seeding`` produces the identical word stream (pinned in
  ``tests/test_cases.py`` against the reference's published stream heads), so
  the generator here is numpy's, about 10x faster than a Python twister.
* :class:`CaseSpec` / :func:`generate_case` -- reference ``oracle.py:111-157``.
* ``config_*`` -- the five BASELINE.json configurations.  No
  public dataset is involved; all inputs are seeded synthetic words.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .keys import KEY_KINDS

__all__ = ["MT19937", "mt19937_next", "CaseSpec", "generate_case", "mt_words",
           "config1", "config2", "config3", "config4", "config5", "CONFIGS"]


class MT19937:
    """Seeded MT19937 word stream (oracle.py:34-108 semantics)."""

    def __init__(self, seed: int):
        self.seed(seed)

    def seed(self, seed: int) -> None:
        bg = np.random.MT19937()
        bg._legacy_seeding(int(seed) & 0xFFFFFFFF)
        self._bg = bg
        self._drawn = 0

    @property
    def index(self) -> int:
        """Position inside the current 624-word block (624 = block exhausted)."""
        return 624 if self._drawn == 0 else ((self._drawn - 1) % 624) + 1

    def next_u32(self) -> int:
        self._drawn += 1
        return int(self._bg.random_raw())

    def draw(self, count: int) -> np.ndarray:
        self._drawn += count
        if count <= 0:
            return np.empty(0, dtype=np.uint32)
        return self._bg.random_raw(count).astype(np.uint32)


def mt19937_next(state: MT19937) -> int:
    return state.next_u32()


def mt_words(seed: int, count: int) -> np.ndarray:
    """First ``count`` words of MT19937(seed) as uint32."""
    return MT19937(seed).draw(count)


@dataclass(frozen=True)
class CaseSpec:
    """One reproducible case: size, key kind, seed (oracle.py:111-128)."""

    size: int
    key_kind: str
    seed: int

    def __post_init__(self):
        if self.size < 0:
            raise ValueError("size must be >= 0")
        if self.key_kind not in KEY_KINDS:
            raise ValueError(f"unknown key kind {self.key_kind!r}")


def generate_case(spec: CaseSpec):
    """Deterministic test sequence (oracle.py:131-157 layouts).

    64-bit kinds take two words per value, high word first; signed32 is a
    reinterpretation of the u32 stream; byte strings are length = w % 17 then
    one byte 1 + w % 255 per position.
    """
    gen = MT19937(spec.seed)
    n = spec.size
    if spec.key_kind == "unsigned32":
        return gen.draw(n)
    if spec.key_kind == "signed32":
        return gen.draw(n).view(np.int32)
    if spec.key_kind in ("unsigned64", "float64"):
        w = gen.draw(2 * n).astype(np.uint64)
        u = (w[0::2] << np.uint64(32)) | w[1::2]
        return u if spec.key_kind == "unsigned64" else u.view(np.float64)
    out = []
    for _ in range(n):
        length = gen.next_u32() % 17
        out.append(bytes(1 + gen.next_u32() % 255 for _ in range(length)))
    return out


# ---------------------------------------------------------------------------
# BASELINE.json configurations
# ---------------------------------------------------------------------------

def config1(n: int = 1 << 20) -> np.ndarray:
    """cfg1: first n words of MT19937(0) as u32 (the reference oracle run)."""
    return generate_case(CaseSpec(n, "unsigned32", 0))


def config2(n: int = 1 << 28) -> np.ndarray:
    """cfg2: n words of MT19937(1) as u32."""
    return mt_words(1, n)


def config3(dist: str, n: int = 1 << 28) -> np.ndarray:
    """cfg3: u64 keys from seed 2; dist in {"uniform", "zipf", "low16"}.

    * uniform: generate_case(CaseSpec(n, 'unsigned64', 2)) (high word first);
    * low16:   the uniform words & 0xFFFF (top 48 bits zero);
    * zipf:    Zipf(s=1.1) over 2^20 distinct u64 values, defined for this
      build (the reference has no such generator): rng = default_rng(2);
      V = 2^20 distinct draws of rng.integers(0, 2^64) (deduplicated, then
      permuted); rank r in [1, 2^20] with P ~ r^-1.1 by inverse CDF over
      rng.random(n); key = V[rank-1].
    """
    if dist == "uniform":
        return generate_case(CaseSpec(n, "unsigned64", 2))
    if dist == "low16":
        return generate_case(CaseSpec(n, "unsigned64", 2)) & np.uint64(0xFFFF)
    if dist == "zipf":
        rng = np.random.default_rng(2)
        nv = 1 << 20
        vals = np.unique(rng.integers(0, np.iinfo(np.uint64).max, size=nv + nv // 8,
                                      dtype=np.uint64, endpoint=True))
        vals = rng.permutation(vals)[:nv]
        assert vals.size == nv
        w = np.arange(1, nv + 1, dtype=np.float64) ** -1.1
        cdf = np.cumsum(w)
        cdf /= cdf[-1]
        out = np.empty(n, dtype=np.uint64)
        step = 1 << 24
        for s in range(0, n, step):
            m = min(step, n - s)
            r = np.searchsorted(cdf, rng.random(m), side="right")
            np.minimum(r, nv - 1, out=r)
            out[s:s + m] = vals[r]
        return out
    raise ValueError(f"unknown cfg3 distribution {dist!r}")


def config4(n: int = 1 << 28) -> tuple[np.ndarray, np.ndarray]:
    """cfg4: KV pairs from one MT19937(3) stream.

    V = the first 1024 distinct u32 words in stream order; the next n words
    w_i give key_i = V[w_i mod 1024]; payload p_i = i (u32).
    """
    gen = MT19937(3)
    seen: dict[int, None] = {}
    while len(seen) < 1024:
        for w in gen.draw(1024 - len(seen)):
            if len(seen) < 1024:
                seen.setdefault(int(w), None)
    V = np.fromiter(seen.keys(), dtype=np.uint32, count=1024)
    w = gen.draw(n)
    keys = V[w & np.uint32(1023)]
    payload = np.arange(n, dtype=np.uint32)
    return keys, payload


def config5(kind: str = "uniform", n: int = 1 << 30) -> np.ndarray:
    """cfg5: n words of MT19937(4) as u32; kind in {"uniform", "sorted", "reverse"}."""
    x = mt_words(4, n)
    if kind == "uniform":
        return x
    x.sort()
    if kind == "sorted":
        return x
    if kind == "reverse":
        return x[::-1].copy()
    raise ValueError(f"unknown cfg5 kind {kind!r}")


CONFIGS = {
    "cfg1": lambda n=None: config1(n or 1 << 20),
    "cfg2": lambda n=None: config2(n or 1 << 28),
    "cfg3_uniform": lambda n=None: config3("uniform", n or 1 << 28),
    "cfg3_zipf": lambda n=None: config3("zipf", n or 1 << 28),
    "cfg3_low16": lambda n=None: config3("low16", n or 1 << 28),
    "cfg4": lambda n=None: config4(n or 1 << 28),
    "cfg5": lambda n=None: config5("uniform", n or 1 << 30),
    "cfg5_sorted": lambda n=None: config5("sorted", n or 1 << 30),
    "cfg5_reverse": lambda n=None: config5("reverse", n or 1 << 30),
}
