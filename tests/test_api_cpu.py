"""Host-side API behaviour that needs no GPU: codecs, contracts, errors, routing."""

import math
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

import paper_0811_3448_b200 as bs
from paper_0811_3448_b200 import keys
from paper_0811_3448_b200.core import Metrics, SortRange


def test_public_surface_mirrors_reference():
    for name in ("sort", "partition", "binar_sort_range", "Metrics", "SortRange", "PartitionResult",
                 "UnsignedCodec", "SignedCodec", "Float64Codec", "ByteStringCodec", "KeyCodec",
                 "codec_for_kind", "sort_iterative", "sort_optimized", "sort_parallel",
                 "OptimizationConfig", "MT19937", "CaseSpec", "generate_case", "BACKEND",
                 "msb_mask", "bit_at_unsigned", "encode_signed", "decode_signed",
                 "encode_float_total_order", "decode_float_total_order", "bit_at_bytestring"):
        assert hasattr(bs, name), name
    assert bs.BACKEND == "cuda"


def test_bit_helpers():
    # keys.py:40-48 examples (SPEC bit_at_unsigned)
    assert keys.bit_at_unsigned(0xB, 0, 4) == 1
    assert keys.bit_at_unsigned(0x7, 0, 4) == 0
    assert keys.bit_at_unsigned(0, 3, 8) == 0
    with pytest.raises(AssertionError):
        keys.bit_at_unsigned(1, 4, 4)
    assert keys.bit_at_bytestring(b"\x80", 0) == 1 and keys.bit_at_bytestring(b"", 3) == 0


def test_signed_codec_exhaustive_width8():
    vals = list(range(-128, 128))
    enc = [keys.encode_signed(v, 8) for v in vals]
    assert enc == sorted(enc) and len(set(enc)) == 256
    assert [keys.decode_signed(u, 8) for u in enc] == vals
    assert keys.encode_signed(0, 32) == 0x80000000 and keys.encode_signed(-1, 32) == 0x7FFFFFFF


def test_float_total_order():
    # tests/test_keys.py: -inf < -3.25 < -0.0 < 0.0 < 1.5 < inf, NaNs at the extremes
    xs = [-math.inf, -3.25, -0.0, 0.0, 1.5, math.inf]
    enc = [keys.encode_float_total_order(keys.double_to_bits(x), 64) for x in xs]
    assert enc == sorted(enc) and len(set(enc)) == len(enc)
    nan_pos = struct.unpack("<Q", struct.pack("<d", float("nan")))[0]
    nan_neg = nan_pos | (1 << 63)
    assert keys.encode_float_total_order(nan_neg, 64) < enc[0]
    assert keys.encode_float_total_order(nan_pos, 64) > enc[-1]
    for b in (0, 1 << 63, nan_pos, nan_neg, keys.double_to_bits(2.5)):
        assert keys.decode_float_total_order(keys.encode_float_total_order(b, 64), 64) == b


def test_words_view_compat():
    a = np.array([-3, 5, -1], dtype=np.int32)
    words, restore = keys.SignedCodec(32).words_view(a)
    assert words.dtype == np.uint32 and words[0] == keys.encode_signed(-3, 32)
    restore()
    assert a.tolist() == [-3, 5, -1]
    f = np.array([-1.5, 0.0, 2.0])
    words, restore = keys.Float64Codec().words_view(f)
    assert words[1] == 1 << 63
    restore()
    assert f.tolist() == [-1.5, 0.0, 2.0]
    assert keys.UnsignedCodec(32).words_view([1, 2]) is None


def test_codec_validation():
    with pytest.raises(ValueError):
        keys.UnsignedCodec(0)
    with pytest.raises(ValueError):
        keys.UnsignedCodec(65)
    with pytest.raises(ValueError):
        keys.SignedCodec(1)
    with pytest.raises(ValueError):
        keys.codec_for_kind("nope")
    with pytest.raises(ValueError):
        keys.ByteStringCodec(-1)
    assert keys.ByteStringCodec().width_for([b"ab", b"abcd"]) == 32


def test_gpu_routing():
    assert keys.UnsignedCodec(32).gpu_spec(np.zeros(3, np.uint32)) == 0
    assert keys.SignedCodec(32).gpu_spec(np.zeros(3, np.int32)) == 1
    assert keys.Float64Codec().gpu_spec(np.zeros(3)) == 2
    assert keys.ByteStringCodec().gpu_spec([b"a"]) is None


def test_metrics_merge_and_range_contracts():
    m = Metrics(1, 2, 3, 4)
    m.merge(Metrics(10, 20, 30, 2))
    assert m == Metrics(11, 22, 33, 4)
    with pytest.raises(AssertionError):
        SortRange(-1, 3)
    with pytest.raises(AssertionError):
        SortRange(3, 1)
    assert SortRange(2, 1).is_empty()


def test_trivial_inputs_return_zero_metrics_without_device():
    # core.py:207-212: nothing to do, no launch
    for seq in ([], [5], np.zeros(1, np.uint32)):
        assert bs.sort(seq, keys.UnsignedCodec(8)) == Metrics()
    assert bs.sort_parallel([7], keys.UnsignedCodec(8), 3) == Metrics()
    with pytest.raises(ValueError):
        bs.sort_parallel([1, 2], keys.UnsignedCodec(4), 0)
    with pytest.raises(ValueError):
        bs.OptimizationConfig(sortedness_check_after=-1)


def test_partition_contract_violations_assert():
    # tests/test_core.py:95-101 -- checked before any device work
    with pytest.raises(AssertionError):
        bs.partition([1, 2], SortRange(1, 0, 0), keys.UnsignedCodec(4), Metrics())
    with pytest.raises(AssertionError):
        bs.partition([1, 2], SortRange(0, 1, 4), keys.UnsignedCodec(4), Metrics())
    with pytest.raises(AssertionError):
        bs.partition([1, 2], SortRange(0, 5, 0), keys.UnsignedCodec(4), Metrics())


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError):
        bs.sort(np.array([3, 1, 2], dtype=np.uint32), keys.UnsignedCodec(32))


def test_generic_engine_inputs_rejected():
    class Tagged(keys.KeyCodec):
        width = 4

    with pytest.raises(TypeError):
        bs.sort([(1, "a"), (0, "b")], Tagged())
    with pytest.raises(TypeError):
        bs.sort([b"b", b"a"], keys.ByteStringCodec())


def test_rejects_unknown_backend_env():
    # tests/test_kernels.py:84-91 pattern: bad BINARSORT_BACKEND fails at import
    env = dict(os.environ, BINARSORT_BACKEND="bogus")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    proc = subprocess.run([sys.executable, "-c", "import paper_0811_3448_b200.kernels"],
                          env=env, capture_output=True, text=True, cwd=root)
    assert proc.returncode != 0 and "BINARSORT_BACKEND" in proc.stderr
