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
    # the multi-device entry point fails loudly too (no device to shard over)
    with pytest.raises((qb.BackendError, ValueError)):
        _lib.solve_devices(np.eye(4), [0, 1])


def test_version_string():
    assert b"sm_100a" in _lib.lib().qb_version()


def _build_c_example(tmp_path):
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = tmp_path / "qb_solve_example"
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", _lib.os.path.join(_lib.REPO_DIR, "include"),
                    _lib.os.path.join(_lib.REPO_DIR, "examples", "qb_solve_example.c"), "-L", _lib.PKG_DIR,
                    "-lqubrute_b200", f"-Wl,-rpath,{_lib.PKG_DIR}", "-o", str(exe)], check=True)
    return exe


def test_plain_c_consumer_builds_and_reports_no_device(tmp_path, cuda_available):
    """The C ABI is usable from C alone (header + .so); without a GPU it reports QB_E_NODEV (exit 2)."""
    import subprocess

    exe = _build_c_example(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert "eval_upper worked example = 2" in out.stdout
    if not cuda_available:
        assert out.returncode == 2 and "no CUDA device" in out.stdout


@pytest.mark.gpu
def test_plain_c_consumer_solves_on_gpu(tmp_path):
    import subprocess

    exe = _build_c_example(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    lines = {l.split(" min ")[0]: l for l in out.stdout.splitlines() if " min " in l}
    # the same instance through the oracle: the C program's SplitMix64 stream (seed 12345)
    from paper_2310_19373_b200 import instances

    n = 24
    u = instances._u64_stream(12345, n * (n + 1) // 2)
    c = np.zeros((n, n))
    c[np.triu_indices(n)] = (u % np.uint64(201)).astype(np.int64) - 100
    bits, val, _ = O.expected_argmin(c, 0)
    assert f"min {val:.1f} argmin {hex(bits)}" in lines["n=24"]
    bits3, val3, _ = O.expected_argmin(c, 3)
    assert f"min {val3:.1f} argmin {hex(bits3)}" in lines["2 shards, m=3:"]
