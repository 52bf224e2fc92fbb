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
    return sorted(set(re.findall(r"\b(qb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert _declared_symbols() == sorted(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared_symbols():
        assert hasattr(L, name), name


def test_result_struct_layout():
    assert ctypes.sizeof(_lib.QbResult) == 136
    assert _lib.QbResult.exact_blocks.offset == 128
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


def _text_sections(img: bytes):
    import struct

    shoff = struct.unpack_from("<Q", img, 0x28)[0]
    shentsize, shnum, shstrndx = struct.unpack_from("<HHH", img, 0x3A)
    secs = [struct.unpack_from("<IIQQQQIIQQ", img, shoff + i * shentsize) for i in range(shnum)]
    stroff = secs[shstrndx][4]
    for s in secs:
        o = stroff + s[0]
        name = img[o:img.index(b"\0", o)].decode()
        if name.startswith(".text."):
            yield name, s[4], s[5]


@pytest.mark.parametrize("kind,L", [(1, 10), (1, 14), (1, 20), (1, 22), (2, 12), (2, 20), (2, 22)])
def test_imm_cubin_patches_every_placeholder(kind, L, tmp_path):
    """QB_VARIANT_IMM: the embedded cubin for chunk length L has each of the 512 coarse-table
    placeholder immediates exactly once; the patched image carries the instance's words in exactly
    those instruction slots (IMAD / VIADDMNMX immediates) and no placeholder survives.  Host only."""
    import struct
    import subprocess

    rng = np.random.default_rng(L)
    # packed biased u16 fields as the host builds them (< 2^15 each)
    nw = 512 * kind
    words = (rng.integers(0, 1 << 15, nw) | (rng.integers(0, 1 << 15, nw) << 16)).astype(np.uint32)
    img = _lib.imm_image(L, words, kind)
    sections = list(_text_sections(img))
    assert len(sections) == 1
    name, off, size = sections[0]
    assert (f"ELi{L}ELi128ELb1E" if kind == 1 else f"coarse2_kernelILi5ELi5ELi{L}ELi128E") in name
    seen = {}
    for at in range(off, off + size, 16):
        v = struct.unpack_from("<I", img, at + 4)[0]
        assert (v >> 16) != 0x7A5C or v in set(int(w) for w in words), "placeholder left unpatched"
        op = struct.unpack_from("<H", img, at)[0] & 0xFFF
        if op in (0x424, 0x846, 0x431, 0x802):
            seen[v] = seen.get(v, 0) + 1
    for w in words:
        assert seen.get(int(w), 0) >= 1
    # the SASS disassembles and shows the words as immediates of IMAD / VIADDMNMX
    path = tmp_path / "imm.cubin"
    path.write_bytes(img)
    sass = subprocess.run(["cuobjdump", "-sass", str(path)], capture_output=True, text=True).stdout
    imms = set(int(h, 16) for h in re.findall(r"(?:IMAD|VIADDMNMX\.U16x2)(?:\.MOV\.U32)? R\d+, R\w+(?:\.reuse)?, (?:R\w+(?:\.reuse)?, )?0x([0-9a-f]+)", sass))
    assert sum(int(w) in imms for w in words) >= nw - 20


@pytest.mark.parametrize("kind,L", [(3, 10), (3, 20), (4, 12), (4, 20), (5, 10), (5, 12), (5, 20), (6, 14), (6, 20), (6, 22), (7, 13), (7, 20)])
def test_byte_kernel_cubin_patches_every_placeholder(kind, L):
    """QB_VARIANT_IMM8 / IMM8S / IMM8A / IMM8AS (kinds 3..7): every placeholder of the embedded cubin is
    replaced by the instance's packed byte word (IMAD / IADD3 / UIADD3 immediates) and none survives.
    Host only."""
    import struct

    nw = _lib.IMM_WORDS[kind]
    rng = np.random.default_rng(100 * kind + L)
    words = rng.integers(0, 1 << 32, nw, dtype=np.uint64).astype(np.uint32)
    words[(words >> 16) == 0x7A5C] = 1  # keep the test words distinguishable from placeholders
    img = _lib.imm_image(L, words, kind)
    (name, off, size), = list(_text_sections(img))
    nx = {4: 1, 6: 1, 7: 2}.get(kind, 0)
    fam = "coarse8s_kernel" if nx else "coarse8_kernel"
    assert f"{fam}ILi5ELi5ELi4ELi6ELi{L}ELi128ELb{int(kind >= 5)}E" + (f"Li{nx}ELb0E" if nx else "") in name
    import bench

    assert name == ".text." + bench.imm_symbol(L, kind)  # the symbol bench.py hashes is the one in the cubin
    found = set()
    want = set(int(w) for w in words)
    for at in range(off, off + size, 16):
        v = struct.unpack_from("<I", img, at + 4)[0]
        assert (v >> 16) != 0x7A5C, "placeholder left unpatched"
        if struct.unpack_from("<H", img, at)[0] & 0xFFF in (0x424, 0x810, 0x836, 0x890) and v in want:
            found.add(v)
    assert found == want
