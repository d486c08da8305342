"""Input generators (paper_0811_3448_b200.cases) vs the reference's MT19937 and layouts."""

import numpy as np
import pytest

from paper_0811_3448_b200 import cases
from paper_0811_3448_b200.cases import MT19937, CaseSpec, generate_case


def test_mt19937_heads_match_reference(golden):
    # reference oracle.MT19937 (oracle.py:34-108); tests/test_oracle.py:10-17
    for seed, head in golden["mt19937_heads"].items():
        assert MT19937(int(seed)).draw(12).tolist() == head


def test_mt19937_piecewise_draw_equivalence():
    a = MT19937(1).draw(2000)
    g = MT19937(1)
    b = np.concatenate([g.draw(5), g.draw(619), g.draw(1), g.draw(1375)])
    assert np.array_equal(a, b)
    g = MT19937(1)
    assert [g.next_u32() for _ in range(3)] == a[:3].tolist()


def test_generate_case_layouts(golden):
    # oracle.py:131-157: u64 = two words high first; i32 reinterprets u32
    for kind, words in golden["generate_case_seed7_n9"].items():
        c = generate_case(CaseSpec(9, kind, 7))
        view = c.view({4: np.uint32, 8: np.uint64}[c.itemsize])
        assert view.tolist() == words, kind


def test_casespec_validation():
    with pytest.raises(ValueError):
        CaseSpec(-1, "unsigned32", 0)
    with pytest.raises(ValueError):
        CaseSpec(3, "nope", 0)


def test_bytestring_generation_shape():
    v = generate_case(CaseSpec(50, "bytestring", 3))
    assert len(v) == 50 and all(isinstance(s, bytes) and len(s) <= 16 and 0 not in s for s in v)


def test_config_generators_small():
    assert cases.config1(16).dtype == np.uint32
    x2 = cases.config2(1000)
    assert x2.dtype == np.uint32 and np.array_equal(x2, cases.mt_words(1, 1000))
    u = cases.config3("uniform", 1000)
    assert u.dtype == np.uint64
    lo = cases.config3("low16", 1000)
    assert int(lo.max()) <= 0xFFFF and np.array_equal(lo, u & np.uint64(0xFFFF))
    z = cases.config3("zipf", 1 << 16)
    assert z.dtype == np.uint64 and np.unique(z).size < z.size
    k, p = cases.config4(1 << 14)
    assert k.dtype == np.uint32 and np.array_equal(p, np.arange(1 << 14, dtype=np.uint32))
    assert np.unique(k).size <= 1024
    s = cases.config5("sorted", 1 << 12)
    r = cases.config5("reverse", 1 << 12)
    assert np.all(s[1:] >= s[:-1]) and np.array_equal(r, s[::-1])
