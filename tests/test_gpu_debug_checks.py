"""The parity corpus against the bounds-checked build (libbinarsort_b200_debug.so,
-DBS_DEBUG_CHECKS): every global and staging write of the sort kernels checks
its index and reports a violation through bs_sort_status, which the shim turns
into SortOverflowError -- so these runs pass only if no write ever left its
range.  (compute-sanitizer is closed on this GPU pool; this replaces it.)"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(cmd, timeout):
    env = dict(os.environ, BS_LIBRARY="debug")
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, (p.stdout[-3000:], p.stderr[-3000:])
    return p.stdout


@pytest.mark.timeout(900)
def test_checked_build_kernel_families(cuda):
    out = _run([sys.executable, "tools/sanitize_cases.py"], 600)
    assert "checked build loaded" in out and "ALL OK" in out


@pytest.mark.timeout(1500)
def test_checked_build_parity_corpus(cuda):
    from paper_0811_3448_b200 import _lib

    assert os.path.exists(_lib.SO_DEBUG_PATH), "checked build missing"
    out = _run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                "tests/test_gpu_parity.py", "tests/test_gpu_robust.py", "tests/test_gpu_dist.py",
                "-k", "not full_size and not cfg5 and not two_processes and not bench_two_ranks"], 1400)
    assert " passed" in out and "failed" not in out
