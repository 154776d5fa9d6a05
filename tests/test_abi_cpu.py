"""CPU-only checks of the boundary: the library loads, exports exactly what include/molr_b200.h
declares, the ctypes table matches, and the host-side validation mirrors the reference."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "molr_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(molr_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    fns = header_functions()
    for name in ("molr_ctx_create", "molr_cache_create", "molr_score", "molr_mol_top_k", "molr_h_indexer",
                 "molr_two_stage_top_k", "molr_quantize_rows", "molr_nth_largest", "molr_merge_top_k"):
        assert name in fns


def test_library_exports_every_declared_symbol():
    from paper_2306_04039_b200 import _lib as L

    lib = L.load()
    for name in header_functions():
        assert hasattr(lib, name), f"{name} declared in the header but not exported"


def test_ctypes_table_matches_header():
    from paper_2306_04039_b200 import _lib as L

    assert sorted(L.SIGNATURES) == header_functions()


def test_header_argument_counts_match_ctypes():
    from paper_2306_04039_b200 import _lib as L

    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for name, argtypes in L.SIGNATURES.items():
        m = re.search(rf"\b{name}\s*\(([^)]*)\)", src)
        args = [a for a in m.group(1).split(",") if a.strip() and a.strip() != "void"]
        assert len(args) == len(argtypes), name


def test_version_string():
    from paper_2306_04039_b200 import _lib as L

    assert b"sm_100a" in L.load().molr_version()


def test_no_cuda_device_fails_loudly():
    """Without a GPU the first compute call raises; nothing silently runs on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2306_04039_b200 import errors
    from paper_2306_04039_b200.quant import quantize_rowwise

    with pytest.raises(errors.DeviceError):
        quantize_rowwise(np.ones((2, 4), dtype=np.float32))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2306_04039_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            assert "oracle" not in re.sub(r"#.*", "", open(os.path.join(pkg, f)).read()).replace(
                "oracle/", ""), f


def test_hindexer_config_validation_mirrors_reference():
    from paper_2306_04039_b200.errors import OutOfRangeError
    from paper_2306_04039_b200.hindexer import HIndexerConfig

    with pytest.raises(ValueError):
        HIndexerConfig(k_prime=10)
    with pytest.raises(ValueError):
        HIndexerConfig(k_prime=10, lam=5, sample_ratio=0.5)
    with pytest.raises(ValueError):
        HIndexerConfig(k_prime=0, lam=5)
    with pytest.raises(ValueError):
        HIndexerConfig(k_prime=3, lam=5, comparator="bogus")
    with pytest.raises(OutOfRangeError):
        HIndexerConfig(k_prime=100, lam=10).resolve_lambda(50)
    assert HIndexerConfig(k_prime=1, sample_ratio=0.001).resolve_lambda(100) == 1
    # Python banker's rounding (hindexer.py:62): 0.5 * 5 = 2.5 -> 2
    assert HIndexerConfig(k_prime=1, sample_ratio=0.5).resolve_lambda(5) == 2


def test_mol_config_and_mlp_validation():
    from paper_2306_04039_b200.errors import DimensionMismatchError
    from paper_2306_04039_b200.mol import GatingNetwork, Mlp, MoLConfig

    with pytest.raises(ValueError):
        MoLConfig(k_u=0, k_x=1, d=1)
    with pytest.raises(ValueError):
        MoLConfig(k_u=1, k_x=1, d=1, tau=0.5)
    assert MoLConfig(8, 8, 64).num_logits == 64
    with pytest.raises(DimensionMismatchError):
        Mlp(np.zeros((3, 4)), np.zeros(5), np.zeros((4, 2)))
    m = Mlp(np.zeros((3, 4)), np.zeros(4), np.zeros((4, 6)))
    c = Mlp(np.zeros((6, 4)), np.zeros(4), np.zeros((4, 5)))
    with pytest.raises(DimensionMismatchError):
        GatingNetwork(m, m, c)


def test_candidate_and_quant_validation_before_any_device_call():
    from paper_2306_04039_b200.errors import DimensionMismatchError, LengthOverflowError, OutOfRangeError
    from paper_2306_04039_b200.hindexer import nth_largest
    from paper_2306_04039_b200.quant import MAX_DOT_LENGTH, QuantizedRows, int8_dot

    with pytest.raises(LengthOverflowError):
        QuantizedRows(codes=np.zeros((1, MAX_DOT_LENGTH + 1), dtype=np.int8), scales=np.ones(1, dtype=np.float32))
    with pytest.raises(DimensionMismatchError):
        int8_dot(np.ones(3, dtype=np.int8), np.ones(4, dtype=np.int8))
    with pytest.raises(LengthOverflowError):
        big = np.ones(MAX_DOT_LENGTH + 1, dtype=np.int8)
        int8_dot(big, big)
    with pytest.raises(OutOfRangeError):
        nth_largest([1.0, 2.0], 0)
    with pytest.raises(OutOfRangeError):
        nth_largest([1.0, 2.0], 3)
