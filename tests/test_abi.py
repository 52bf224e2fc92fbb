"""CPU-side checks of the native boundary: the library loads without a GPU, exports every
symbol include/qubrute_b200.h declares, and its host-only functions work."""

import ctypes
import re

import numpy as np
import pytest

import paper_2310_19373_b200 as qb
from oracle import oracle as O
from paper_2310_19373_b200 import _lib


def _declared_symbols():
    text = open(_lib.HEADER).read()
    return sorted(set(re.findall(r"\b(qb_[a-z_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert _declared_symbols() == sorted(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared_symbols():
        assert hasattr(L, name), name


def test_result_struct_layout():
    assert ctypes.sizeof(_lib.QbResult) == 112
    assert _lib.QbResult.kernel_ms.offset == 64


def test_eval_upper_matches_oracle_bitwise():
    rng = np.random.default_rng(3)
    for n in (1, 7, 24, 40):
        c = np.triu(rng.standard_normal((n, n)))
        for _ in range(5):
            x = rng.integers(0, 2, n).astype(np.float64)
            assert _lib.eval_upper(c, x) == O.eval_upper(c, x)


def test_evaluate_validation_messages():
    inst = qb.QuboInstance(np.eye(3))
    with pytest.raises(ValueError, match="shape"):
        qb.evaluate(inst, [1, 0])
    with pytest.raises(ValueError, match="0 or 1"):
        qb.evaluate(inst, [1, 2, 0])


def test_no_silent_cpu_fallback_without_gpu(cuda_available):
    if cuda_available:
        pytest.skip("GPU present")
    with pytest.raises(qb.BackendError):
        qb.solve_incremental(qb.QuboInstance(np.eye(4)))


def test_version_string():
    assert b"sm_100a" in _lib.lib().qb_version()
