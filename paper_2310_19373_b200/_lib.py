"""ctypes binding of libqubrute_b200.so (C ABI in include/qubrute_b200.h).

The shared library is built in-tree by :func:`build` (``nvcc -gencode
arch=compute_100a,code=sm_100a``).  There is no CPU fallback: if the library is
missing or no CUDA device is present, solver calls raise :class:`BackendError`.
Host-only helpers (``eval_upper``) work without a GPU.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("QB_LIB_PATH") or os.path.join(PKG_DIR, "libqubrute_b200.so")
HEADER = os.path.join(REPO_DIR, "include", "qubrute_b200.h")
SOURCES = [os.path.join(PKG_DIR, "csrc", f)
           for f in ("qb_api.cu", "qb_k_table.cu", "qb_k_coarse.cu", "qb_k_fieldwalk.cu", "qb_k_batch.cu", "qb_k_tc.cu",
                     "qb_k_byte8.cu")]
DEPS = [os.path.join(PKG_DIR, "csrc", f) for f in os.listdir(os.path.join(PKG_DIR, "csrc"))] + [HEADER]
# patched-immediate coarse kernels (QB_VARIANT_IMM): one cubin per chunk length, embedded in the .so
IMM_SOURCE = os.path.join(PKG_DIR, "csrc", "qb_k_coarse_imm.cu")
IMM2_SOURCE = os.path.join(PKG_DIR, "csrc", "qb_k_coarse2_imm.cu")
IMM_LS = (10, 11, 12, 13, 14, 16, 18, 20, 22)
IMM2_LS = (12, 13, 14, 16, 18, 20, 22)  # super-block kernel: chunks of >= B + 2 free bits
IMM8_SOURCE = os.path.join(PKG_DIR, "csrc", "qb_k_coarse8_imm.cu")  # byte-packed threshold kernel
IMM8_LS = IMM_LS
IMM8S_LS = IMM2_LS  # its 11-bit super-block form
IMM8Q_LS = (13, 14, 16, 18, 20, 22)  # 12-bit super-blocks: chunks of >= B + 3 free bits
IMM_WORDS = {1: 512, 2: 1024, 3: 256, 4: 512, 5: 256, 6: 512, 7: 1024}  # placeholder immediates per patched kernel kind

QB_OK = 0
QB_E_ARG = -1
QB_E_CAP = -2
QB_E_CUDA = -3
QB_E_NODEV = -4
QB_E_INTERNAL = -5

TIE_GRAY = 0
TIE_INTEGER = 1

VARIANT_AUTO = 0
VARIANT_TABLE = 1
VARIANT_FIELDWALK = 2
VARIANT_COARSE = 3
VARIANT_TC = 4
VARIANT_IMM = 5
VARIANT_IMM2 = 6
VARIANT_IMM8 = 7
VARIANT_IMM8S = 8
VARIANT_IMM8A = 9
VARIANT_IMM8AS = 10
VARIANT_IMM8AQ = 11
VARIANT_BYTE8 = 12
# the search kernels AUTO picks among where the coarse filter runs, besides the table-load COARSE: the
# patched-immediate kernels and the table-load byte kernel
IMM_VARIANTS = (VARIANT_IMM, VARIANT_IMM2, VARIANT_IMM8, VARIANT_IMM8S, VARIANT_IMM8A, VARIANT_IMM8AS,
                VARIANT_IMM8AQ, VARIANT_BYTE8)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # -ffp-contract=off: host eval_upper / batch folding keep the reference's fp64 operation order
    # (no FMA contraction), which is what makes the reported values bit-identical
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fopenmp",
    "-shared",
]
LINK_FLAGS = ["-Xcompiler", "-fopenmp"]


class BackendError(RuntimeError):
    """The CUDA backend is unavailable or a kernel failed (never silently falls back)."""


class QbResult(ctypes.Structure):
    _fields_ = [
        ("argmin_bits", ctypes.c_uint64),
        ("value", ctypes.c_double),
        ("tie_key", ctypes.c_uint64),
        ("value_key", ctypes.c_uint64),
        ("states", ctypes.c_uint64),
        ("exact", ctypes.c_int32),
        ("variant", ctypes.c_int32),
        ("scale_exp", ctypes.c_int32),
        ("prefix_bits", ctypes.c_int32),
        ("candidates", ctypes.c_uint64),
        ("kernel_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("search_ms", ctypes.c_double),
        ("collect_ms", ctypes.c_double),
        ("launches", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("param_bytes", ctypes.c_uint64),
        ("module_ms", ctypes.c_double),
        ("combine", ctypes.c_int32),
        ("retries", ctypes.c_int32),
        ("exact_blocks", ctypes.c_uint64),
    ]


_dp = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)

# every symbol include/qubrute_b200.h declares, with its ctypes signature
SIGNATURES = {
    "qb_version": (ctypes.c_char_p, []),
    "qb_last_error": (ctypes.c_char_p, []),
    "qb_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "qb_init": (ctypes.c_int, [ctypes.c_int]),
    "qb_shutdown": (None, []),
    "qb_eval_upper": (ctypes.c_double, [_dp, ctypes.c_int, _dp]),
    "qb_solve": (ctypes.c_int, [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(QbResult)]),
    "qb_solve_devices": (ctypes.c_int, [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(QbResult)]),
    "qb_all_minimisers": (ctypes.c_int, [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, _u64p,
                                         ctypes.c_uint64, _u64p, _dp]),
    "qb_gray_scan": (ctypes.c_int, [_dp, _dp, _dp, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, _dp,
                                    _u64p]),
    "qb_solve_batch": (ctypes.c_int, [_dp, ctypes.c_int, ctypes.c_uint64, _u64p, _dp, _dp]),
    "qb_solve_batch_f32": (ctypes.c_int, [ctypes.POINTER(ctypes.c_float), ctypes.c_int, ctypes.c_uint64, _u64p, _dp,
                                          _dp]),
    "qb_solve_batch_devices": (ctypes.c_int, [_dp, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int),
                                              ctypes.c_int, _u64p, _dp, _dp]),
    "qb_prefix_eval": (ctypes.c_int, [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, _dp, _dp]),
    "qb_imm_image": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_uint32), ctypes.c_char_p,
                                    ctypes.c_uint64, _u64p]),
    "qb_byte_image": (ctypes.c_int, [_dp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_uint32), _dp,
                                     ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)]),
}

_lock = threading.Lock()
_lib = None


def build(force: bool = False, verbose: bool = False, output: str | None = None, defines=()) -> str:
    """Compile libqubrute_b200.so in-tree for sm_100a (skipped when up to date).

    Each translation unit (host runtime + one per kernel family) is compiled by its own nvcc
    process in parallel, then linked with ``nvcc -shared``.  ``output`` / ``defines`` build an
    experimental variant elsewhere (tools/build_variants.sh)."""
    out = output or LIB_PATH
    if not force and output is None and os.path.exists(out):
        mtime = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= mtime for d in DEPS if os.path.exists(d)):
            return out
    objdir = os.path.join(REPO_DIR, "build", "obj", os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + list(defines)
    if not any("-ffp-contract=off" in f for f in compile_flags):
        raise RuntimeError("libqubrute_b200 must be built with -ffp-contract=off (bit-exact host eval_upper)")
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        cmd = ["nvcc", *compile_flags, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd)))
        objs.append(obj)
    cubins = []
    # kinds 3..7: byte-packed threshold kernels (3 + super-block + 2 * row-bound form; 7: row-bound, 12-bit blocks)
    for kind, src, Ls, extra in ((1, IMM_SOURCE, IMM_LS, ()), (2, IMM2_SOURCE, IMM2_LS, ()),
                                  (3, IMM8_SOURCE, IMM8_LS, ()),
                                  (4, IMM8_SOURCE, IMM8S_LS, ("-DQB_IMM8_SUPER=1",)),
                                  (5, IMM8_SOURCE, IMM8_LS, ("-DQB_IMM8_APPROX=1",)),
                                  (6, IMM8_SOURCE, IMM8S_LS, ("-DQB_IMM8_SUPER=1", "-DQB_IMM8_APPROX=1")),
                                  (7, IMM8_SOURCE, IMM8Q_LS, ("-DQB_IMM8_SUPER=2", "-DQB_IMM8_APPROX=1"))):
        for L in Ls:
            cub = os.path.join(objdir, f"qb_coarse_imm{kind}_L{L}.cubin")
            cmd = ["nvcc", *[f for f in compile_flags if not f.startswith("-Xcompiler") and "-fPIC" not in f],
                   f"-DQB_IMM_L={L}", *extra, "-cubin", "-o", cub, src]
            procs.append((f"{src} (L={L})", subprocess.Popen(cmd)))
            cubins.append((kind, L, cub))
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {failed}")
    objs.append(_embed_cubins(objdir, cubins))
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *LINK_FLAGS, "-o", out, *objs],
                   check=True)
    return out


def _embed_cubins(objdir: str, cubins) -> str:
    """C object holding the patched-immediate cubins as byte arrays (qb_imm_cubins[], read by
    qb_api.cu imm_module), compiled with the host C compiler."""
    csrc = os.path.join(objdir, "qb_imm_cubins.c")
    with open(csrc, "w") as fh:
        fh.write("/* generated by paper_2310_19373_b200/_lib.py: patched-immediate coarse cubins */\n")
        fh.write("#include <stddef.h>\n")
        for kind, L, path in cubins:
            data = open(path, "rb").read()
            fh.write(f"static const unsigned char cubin_{kind}_L{L}[{len(data)}] __attribute__((aligned(16))) = {{\n")
            for i in range(0, len(data), 32):
                fh.write(",".join(str(b) for b in data[i:i + 32]) + ",\n")
            fh.write("};\n")
        fh.write("struct qb_imm_cubin { int kind; int L; const unsigned char* data; size_t size; };\n")
        fh.write("const struct qb_imm_cubin qb_imm_cubins[] = {\n")
        for kind, L, path in cubins:
            fh.write(f"  {{{kind}, {L}, cubin_{kind}_L{L}, sizeof(cubin_{kind}_L{L})}},\n")
        fh.write("  {0, 0, 0, 0}};\n")
    obj = csrc.replace(".c", ".o")
    subprocess.run(["cc", "-O1", "-fPIC", "-c", "-o", obj, csrc], check=True)
    return obj


def lib():
    """Load (once) and return the native library; raises BackendError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BackendError(f"{LIB_PATH} not built: run __graft_entry__.build() or "
                                   "python -c 'import paper_2310_19373_b200._lib as l; l.build()'")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def last_error() -> str:
    msg = lib().qb_last_error()
    return msg.decode() if msg else ""


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def eval_upper(coeffs, x) -> float:
    """Host-side eval_upper (_kernels.py:12-20) from the native library."""
    c = _f64(coeffs)
    xv = _f64(x)
    return float(lib().qb_eval_upper(_ptr(c), c.shape[0], _ptr(xv)))


def device_count() -> int:
    c = ctypes.c_int(0)
    lib().qb_device_count(ctypes.byref(c))
    return c.value


def default_device() -> int:
    return int(os.environ.get("QB_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def init(device: int | None = None) -> None:
    dev = default_device() if device is None else device
    rc = lib().qb_init(dev)
    if rc != QB_OK:
        raise BackendError(f"qb_init({dev}) failed: {last_error()}")


def check(rc: int, what: str) -> None:
    if rc == QB_OK:
        return
    msg = last_error()
    if rc == QB_E_CAP:
        from .core import DimensionCapError

        raise DimensionCapError(msg)
    if rc == QB_E_ARG:
        raise ValueError(msg)
    raise BackendError(f"{what} failed ({rc}): {msg}")


def solve(coeffs, m_fix: int = 0, suffix: int = 0, m_tie: int = 0, tie_rule: int = TIE_GRAY, shard: int = 0,
          shard_count: int = 1, variant: int = VARIANT_AUTO, device: int | None = None) -> QbResult:
    c = _f64(coeffs)
    init(device)
    out = QbResult()
    rc = lib().qb_solve(_ptr(c), c.shape[0], m_fix, suffix, m_tie, tie_rule, shard, shard_count, variant,
                        ctypes.byref(out))
    check(rc, "qb_solve")
    return out


def solve_devices(coeffs, devices, m_fix: int = 0, suffix: int = 0, m_tie: int = 0, tie_rule: int = TIE_GRAY,
                  variant: int = VARIANT_AUTO) -> QbResult:
    """One solve sharded over several GPUs of this process (qb_solve_devices): shard i on devices[i]."""
    c = _f64(coeffs)
    devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
    out = QbResult()
    rc = lib().qb_solve_devices(_ptr(c), c.shape[0], m_fix, suffix, m_tie, tie_rule, devs, len(devices), variant,
                                ctypes.byref(out))
    check(rc, "qb_solve_devices")
    return out


def all_minimisers(coeffs, m_fix: int = 0, suffix: int = 0, m_tie: int = 0, cap: int = 1 << 20,
                   device: int | None = None):
    """(value, uint64 array of every minimiser sorted by the Gray tie rule, total count)."""
    c = _f64(coeffs)
    init(device)
    out = np.zeros(max(cap, 1), dtype=np.uint64)
    cnt = ctypes.c_uint64()
    val = ctypes.c_double()
    rc = lib().qb_all_minimisers(_ptr(c), c.shape[0], m_fix, suffix, m_tie, out.ctypes.data_as(_u64p), cap,
                                 ctypes.byref(cnt), ctypes.byref(val))
    check(rc, "qb_all_minimisers")
    return val.value, out[: min(cap, cnt.value)].copy(), int(cnt.value)


def gray_scan(coeffs, qua, lin, x0, v0, n_free, device: int | None = None):
    c, q, l, x = _f64(coeffs), _f64(qua), _f64(lin), _f64(x0)
    n = c.shape[0]
    init(device)
    xm = np.zeros(n)
    vm = ctypes.c_double()
    steps = ctypes.c_uint64()
    rc = lib().qb_gray_scan(_ptr(c), _ptr(q), _ptr(l), _ptr(x), float(v0), n, int(n_free), _ptr(xm),
                            ctypes.byref(vm), ctypes.byref(steps))
    check(rc, "qb_gray_scan")
    return xm, vm.value, int(steps.value)


def solve_batch(coeffs_batch, device: int | None = None):
    """(argmin bits, values, device window ms) of a (count, n, n) batch; a float32 array goes to
    qb_solve_batch_f32 as it is (no fp64 copy), anything else is converted to fp64."""
    f32 = isinstance(coeffs_batch, np.ndarray) and coeffs_batch.dtype == np.float32
    c = np.ascontiguousarray(coeffs_batch) if f32 else _f64(coeffs_batch)
    count, n = c.shape[0], c.shape[1]
    init(device)
    bits = np.zeros(count, dtype=np.uint64)
    vals = np.zeros(count)
    ms = ctypes.c_double()
    if f32:
        rc = lib().qb_solve_batch_f32(c.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n, count,
                                      bits.ctypes.data_as(_u64p), _ptr(vals), ctypes.byref(ms))
    else:
        rc = lib().qb_solve_batch(_ptr(c), n, count, bits.ctypes.data_as(_u64p), _ptr(vals), ctypes.byref(ms))
    check(rc, "qb_solve_batch")
    return bits, vals, ms.value


def solve_batch_devices(coeffs_batch, devices):
    """The batch split over ``devices`` (qb_solve_batch_devices): slice i of the instances on devices[i]."""
    c = _f64(coeffs_batch)
    count, n = c.shape[0], c.shape[1]
    devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
    bits = np.zeros(count, dtype=np.uint64)
    vals = np.zeros(count)
    ms = ctypes.c_double()
    rc = lib().qb_solve_batch_devices(_ptr(c), n, count, devs, len(devices), bits.ctypes.data_as(_u64p), _ptr(vals),
                                      ctypes.byref(ms))
    check(rc, "qb_solve_batch_devices")
    return bits, vals, ms.value


def prefix_eval(coeffs, k: int, c_begin: int, count: int, device: int | None = None):
    c = _f64(coeffs)
    n = c.shape[0]
    init(device)
    vals = np.zeros(count)
    fields = np.zeros((count, n - k))
    rc = lib().qb_prefix_eval(_ptr(c), n, k, c_begin, count, _ptr(vals), _ptr(fields))
    check(rc, "qb_prefix_eval")
    return vals, fields


def byte_image(coeffs, kind: int):
    """Host-only test hook: (words, quantized upper-triangular Q, fl(1/unit), Rneg, slack, scale_exp) of the byte
    image the threshold kernel of `kind` (3..6) builds for `coeffs` (qb_byte_image)."""
    c = _f64(coeffs)
    n = c.shape[0]
    words = np.zeros(IMM_WORDS[kind], dtype=np.uint32)
    quant = np.zeros((n, n), dtype=np.float64)
    inv, rneg, slack, e = ctypes.c_float(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32()
    check(lib().qb_byte_image(_ptr(c), n, kind, words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), _ptr(quant),
                              ctypes.byref(inv), ctypes.byref(rneg), ctypes.byref(slack), ctypes.byref(e)),
          "qb_byte_image")
    return words, quant, np.float32(inv.value), int(rneg.value), int(slack.value), int(e.value)


def imm_image(L: int, words, kind: int = 1) -> bytes:
    """The patched-immediate cubin of `kind` (1: QB_VARIANT_IMM, 2: IMM2, 3: IMM8, 4: IMM8S, 5: IMM8A,
    6: IMM8AS, 7: IMM8AQ; IMM_WORDS[kind] table words) for chunk length L with coarse table words `words` (test hook)."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    if kind not in IMM_WORDS or w.shape != (IMM_WORDS[kind],):
        raise ValueError(f"kind {kind} needs {IMM_WORDS.get(kind)} table words")
    size = ctypes.c_uint64()
    wp = w.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
    check(lib().qb_imm_image(kind, L, wp, None, 0, ctypes.byref(size)), "qb_imm_image")
    buf = ctypes.create_string_buffer(size.value)
    check(lib().qb_imm_image(kind, L, wp, buf, size.value, ctypes.byref(size)), "qb_imm_image")
    return buf.raw[: size.value]
