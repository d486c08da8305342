"""bench.py's CPU legs and host helpers (no GPU): the reference arm's JSON
line and the order-independent checksum the N>1 correctness check uses."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
                        "--n", str(1 << 20)], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    r = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert r["impl"] == "reference" and r["steps"] == 2 and r["value"] > 0
    assert r["e2e"]["h2d_bytes_per_step"] == 0 and r["e2e"]["value"] == r["value"]
    cb = r["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["checked"] and cb["cores"] >= 1
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "binarsort")):
        assert cb["kind"] == "reference"
    assert r["config"]["same_config"] and r["config"]["global_batch"] == 1 << 20


def test_checksum_is_order_independent_and_sensitive():
    torch = pytest.importorskip("torch")
    sys.path.insert(0, ROOT)
    import bench

    rng = np.random.default_rng(0)
    x = rng.integers(0, 2 ** 32, 10000, dtype=np.uint64).astype(np.uint32)
    a = bench._checksum(torch.from_numpy(x.view(np.int32)))
    b = bench._checksum(torch.from_numpy(np.sort(x).view(np.int32)))
    assert torch.equal(a, b)
    y = x.copy()
    y[0], y[1] = y[1], y[1]  # lose one key, duplicate another
    if x[0] != x[1]:
        assert not torch.equal(a, bench._checksum(torch.from_numpy(y.view(np.int32))))
    # sums of two keys can collide; the mixed sum must not for this swap
    z = x.copy()
    z[0] = z[0] + 1
    z[1] = z[1] - 1
    c = bench._checksum(torch.from_numpy(z.view(np.int32)))
    assert int(c[0]) == int(a[0]) and int(c[1]) != int(a[1])
