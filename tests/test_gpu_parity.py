"""GPU parity: the CUDA path (through the C ABI) against the reference's golden outputs
and the CPU oracle.  Integer instances: bit-exact values and argmins.  Float instances:
argmin exact and value bit-identical (the value is eval_upper of the argmin).  Tie rules:
every entry point's rule, on tie-heavy instances.
"""

import io

import numpy as np
import pytest

import paper_2310_19373_b200 as qb
from oracle import oracle as O
from paper_2310_19373_b200 import _kernels, _lib, instances

pytestmark = pytest.mark.gpu


def _bits(sol):
    return qb.bits_to_int(sol.minimizer)


def _check(sol, want, name):
    assert _bits(sol) == want["bits"], (name, _bits(sol), want["bits"])
    assert sol.value == want["value"], (name, sol.value, want["value"])
    assert sol.evaluations == want["evaluations"], name


def test_golden_cases(golden):
    for case in golden["cases"]:
        inst = qb.QuboInstance(np.array(case["coeffs"]))
        for key, want in case["results"].items():
            name = f"{case['name']}:{key}"
            if key == "incremental":
                _check(qb.solve_incremental(inst), want, name)
            elif key.startswith("parallel_m"):
                m = int(key[len("parallel_m"):])
                _check(qb.solve_parallel(inst, qb.SolveConfig(threads=4, fixed_bits=m)), want, name)
            elif key == "naive":
                _check(qb.solve_naive(inst), want, name)
            elif key.startswith("subspace_m"):
                m = int(key[len("subspace_m"):])
                for s, w in enumerate(want):
                    _check(qb.solve_subspace(inst, qb.SubspaceSpec(m, s)), w, f"{name}:{s}")


def test_gray_scan_seam(golden):
    for case in golden["gray_scan"]:
        c = np.array(case["coeffs"])
        form = qb.split(qb.QuboInstance(c))
        xm, vm, steps = _kernels.gray_scan(c, form.qua, form.lin, np.array(case["x0"]), case["v0"], case["n_free"])
        assert xm.tolist() == case["x_min"]
        assert vm == case["v_min"]
        assert steps == case["steps"]


def _tie_heavy(n, seed, lo=-2, hi=2):
    return instances.int_uniform_coeffs(n, seed, lo, hi)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11, 12, 13, 14])
def test_tie_rules_against_enumeration(n):
    for rep in range(6):
        c = _tie_heavy(n, 1000 * n + rep)
        inst = qb.QuboInstance(c)
        bits, val, _ = O.expected_argmin(c, 0)
        sol = qb.solve_incremental(inst)
        assert _bits(sol) == bits and sol.value == val
        bits, val, _ = O.expected_argmin(c, 0, rule="integer")
        assert _bits(qb.solve_naive(inst)) == bits
        for m in sorted({1, n // 2, n - 1}):
            if not 0 < m < n:
                continue
            bits, val, _ = O.expected_argmin(c, m)
            sol = qb.solve_parallel(inst, qb.SolveConfig(threads=2, fixed_bits=m))
            assert _bits(sol) == bits, (n, rep, m)
            for s in (0, (1 << m) - 1, (1 << m) // 3):
                bits, val, _ = O.expected_argmin(c, m, suffix=s)
                sol = qb.solve_subspace(inst, qb.SubspaceSpec(m, s))
                assert _bits(sol) == bits, (n, rep, m, s)


def test_degenerate_all_tied():
    # zero matrix: every state ties; lowest key is the zero vector for every rule
    for n in (1, 6, 17, 24):
        inst = qb.QuboInstance(np.zeros((n, n)))
        assert _bits(qb.solve_incremental(inst)) == 0
        assert _bits(qb.solve_naive(inst, max_n=40)) == 0
        if n >= 2:
            assert _bits(qb.solve_parallel(inst, qb.SolveConfig(threads=4, fixed_bits=min(2, n - 1)))) == 0
            s = qb.solve_subspace(inst, qb.SubspaceSpec(1, 1))
            assert _bits(s) == 1 << (n - 1)


@pytest.mark.parametrize("n", [18, 20, 22, 24])
def test_medium_sizes_against_enumeration(n):
    for name in ("A", "B", "D", "E"):
        c = instances.config_coeffs(name, 3, n=n)
        bits, val, mins = O.expected_argmin(c, 0)
        sol = qb.solve_incremental(qb.QuboInstance(c))
        assert _bits(sol) == bits, (name, n)
        assert sol.value == O.eval_upper(c, sol.minimizer.astype(np.float64))


def test_random_fp64_instances_vs_oracle():
    # the reference's own generator gives fp64 (non-quantizable) values: certified filter path
    for n in (10, 16, 21):
        for rep in range(3):
            inst = instances.random_instance(n, instances.bench_seed(n, rep))
            bits, val, ev = O.solve_incremental(inst.coeffs)
            sol = qb.solve_incremental(inst)
            assert (_bits(sol), sol.value, sol.evaluations) == (bits, val, ev)
            res = _lib.solve(inst.coeffs)
            assert res.exact == 0 and res.candidates >= 1


def test_config_d_full_golden(golden):
    case = next(c for c in golden["cases"] if c["name"] == "configD_n32_rep0")
    inst = qb.QuboInstance(np.array(case["coeffs"]))
    _check(qb.solve_parallel(inst, qb.SolveConfig(threads=8, fixed_bits=6)), case["results"]["parallel_m6"], "D")
    res = _lib.solve(inst.coeffs)
    assert res.exact == 1


def test_config_b_full_golden(golden):
    case = next(c for c in golden["cases"] if c["name"] == "configB_n24_rep0")
    inst = qb.QuboInstance(np.array(case["coeffs"]))
    _check(qb.solve_incremental(inst), case["results"]["incremental"], "B")


def test_sharding_is_invariant():
    # the chunk space split into S shards and combined by (value_key, tie_key) == one launch
    for name, n in (("D", 28), ("E", 30), ("A", 20)):
        c = instances.config_coeffs(name, 1, n=n)
        whole = _lib.solve(c)
        for S in (2, 3, 8):
            parts = [_lib.solve(c, shard=i, shard_count=S) for i in range(S)]
            best = min(parts, key=lambda r: (r.value_key, r.tie_key))
            assert (best.argmin_bits, best.value, best.tie_key) == (whole.argmin_bits, whole.value, whole.tie_key)
            assert sum(p.states for p in parts) == 1 << n


def test_solve_devices_matches_single_solve():
    """qb_solve_devices (one process, shard i on devices[i], host combine) == one launch; with the one
    GPU here every shard runs on device 0 (the same code path a multi-GPU box runs in parallel)."""
    for name, n in (("D", 30), ("E", 32), ("A", 20)):
        c = instances.config_coeffs(name, 2, n=n)
        whole = _lib.solve(c)
        for ndev in (1, 2, 3):
            r = _lib.solve_devices(c, [0] * ndev)
            assert (r.argmin_bits, r.value, r.tie_key) == (whole.argmin_bits, whole.value, whole.tie_key)
            assert r.states == 1 << n
        r = _lib.solve_devices(c, [0, 0], m_fix=3, suffix=5, m_tie=3)
        w = _lib.solve(c, 3, 5, 3)
        assert (r.argmin_bits, r.value, r.tie_key) == (w.argmin_bits, w.value, w.tie_key)


def test_solver_devices_knob():
    """SolveConfig(devices=...) / solve_incremental(devices=...) shard through qb_solve_devices and
    return the reference's answer (all shards on device 0 here)."""
    c = instances.config_coeffs("D", 4, n=26)
    inst = qb.QuboInstance(c)
    ref_inc = qb.solve_incremental(inst)
    ref_par = qb.solve_parallel(inst, qb.SolveConfig(threads=8))
    got_inc = qb.solve_incremental(inst, devices=(0, 0, 0))
    got_par = qb.solve_parallel(inst, qb.SolveConfig(threads=8, devices=(0, 0)))
    got_dsp = qb.solve(inst, qb.SolveConfig(mode="incremental", devices=(0,)))
    for a, b in ((ref_inc, got_inc), (ref_par, got_par), (ref_inc, got_dsp)):
        assert _bits(a) == _bits(b) and a.value == b.value and a.evaluations == b.evaluations


def test_config_e_n40_properties():
    """n=40 is beyond the oracle: check the argmin against exact CPU scans of the
    subspace that contains it and of random other subspaces; the default (coarse-filter)
    kernel, the fp32 table kernel and the field walk agree."""
    c = instances.config_coeffs("E", 0)
    inst = qb.QuboInstance(c)
    sol = qb.solve_incremental(inst)
    auto = _lib.solve(c)
    assert auto.variant in _lib.IMM_VARIANTS  # n=40: a patched-immediate coarse kernel
    table = _lib.solve(c, variant=_lib.VARIANT_TABLE)
    coarse = _lib.solve(c, variant=_lib.VARIANT_COARSE)
    for other in (table, coarse):
        assert (auto.argmin_bits, auto.value, auto.tie_key) == (other.argmin_bits, other.value, other.tie_key)
    x = _bits(sol)
    assert sol.value == O.eval_upper(c, sol.minimizer.astype(np.float64))
    m = 17  # 2^23-state subspaces
    suffix = x >> (40 - m)
    bits, val, _ = O.solve_subspaces(c, m, suffix, suffix + 1, threads=8)
    assert bits == x and val == sol.value
    rng = np.random.default_rng(0)
    for s in rng.integers(0, 1 << m, size=4):
        _, v, _ = O.solve_subspaces(c, m, int(s), int(s) + 1, threads=8)
        assert v >= sol.value


@pytest.mark.parametrize("rep", [1, 2, 3])
def test_config_e_n40_other_seeds(rep):
    """Config E at n=40 for further seeds: coarse kernel (with its LDC rows), fp32 table kernel and
    tensor-core pass agree, and the argmin is the exact minimum of its own 2^23-state subspace."""
    c = instances.config_coeffs("E", rep)
    auto = _lib.solve(c)
    table = _lib.solve(c, variant=_lib.VARIANT_TABLE)
    tcr = _lib.solve(c, variant=_lib.VARIANT_TC)
    for r in (table, tcr):
        assert (auto.argmin_bits, auto.value, auto.tie_key) == (r.argmin_bits, r.value, r.tie_key)
    x = int(auto.argmin_bits)
    m = 17
    bits, val, _ = O.solve_subspaces(c, m, x >> (40 - m), (x >> (40 - m)) + 1, threads=8)
    assert bits == x and val == auto.value


def test_batch_config_c_golden(golden):
    cb = golden["configC"]
    batch = instances.config_batch(cb["count"], cb["n"])
    bits, vals, ms = _lib.solve_batch(batch)
    assert [int(b) for b in bits] == cb["bits"]
    assert vals.tolist() == cb["values"]
    sols = qb.solve_batch(batch[:64])
    assert [_bits(s) for s in sols] == cb["bits"][:64]


def test_batch_rejects_non_finite():
    """Non-finite coefficients anywhere in a batch (also below the diagonal) raise ValueError like
    QuboInstance does; the check runs in the batch kernel (no host pass over the batch)."""
    batch = instances.config_batch(64, 16)
    for pos in ((5, 3, 7), (63, 9, 2), (0, 0, 0)):
        bad = batch.copy()
        bad[pos] = np.nan if pos != (0, 0, 0) else np.inf
        with pytest.raises(ValueError, match="finite"):
            qb.solve_batch(bad)
    bits, vals, _ = _lib.solve_batch(batch)  # and the device is fine afterwards
    assert len(bits) == 64


@pytest.mark.parametrize("n", [1, 2, 5, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 20])
def test_batch_ties_and_sizes(n):
    count = 40
    batch = np.stack([_tie_heavy(n, 77 * n + b, -1, 1) for b in range(count)])
    batch[3] = 0.0  # all states tied: candidate overflow -> single-instance fallback
    bits, vals, _ = _lib.solve_batch(batch)
    for b in range(count):
        want, wv, _ = O.expected_argmin(batch[b], 0)
        assert int(bits[b]) == want, (n, b)
        assert vals[b] == wv


def test_batch_float_instances_vs_oracle():
    for n in (12, 18):
        batch = np.stack([instances.normal_coeffs(n, 5000 + b) for b in range(24)])
        bits, vals, _ = _lib.solve_batch(batch)
        ob, ov = O.solve_batch(batch, threads=8)
        assert [int(b) for b in bits] == [int(b) for b in ob]
        assert vals.tolist() == ov.tolist()


def test_batch_pipeline_mixed_formats_and_folding():
    """The host packs the batch in pieces (fp32 upper triangle when every folded coefficient is
    fp32-exact, else fp64) and pipelines pack / H2D / kernel.  3000 instances = 4 pieces; one
    piece holds a coefficient that is not fp32-representable (that piece ships fp64), and half of
    the instances carry their off-diagonal weights split between the upper and lower triangle, so
    the host fold (core.py:66-72) is exercised.  Every answer equals the oracle on the folded
    matrices, bit for bit."""
    n, count = 14, 3000
    batch = np.stack([instances.normal_coeffs(n, 9100 + b, density=0.5) for b in range(count)])
    iu = np.triu_indices(n, 1)
    for b in range(0, count, 2):
        half = np.float32(0.5) * batch[b][iu].astype(np.float32)
        batch[b][(iu[1], iu[0])] = half
        batch[b][iu] = batch[b][iu] - half
    batch[1700, 2, 5] += 0.1  # piece 2 (instances 1500..2249) -> fp64 format
    folded = np.stack([qb.QuboInstance(batch[b]).coeffs for b in range(count)])
    bits, vals, _ = _lib.solve_batch(batch)
    ob, ov = O.solve_batch(folded, threads=8)
    assert [int(b) for b in bits] == [int(b) for b in ob]
    assert vals.tolist() == ov.tolist()
    mins, mvals = qb.solve_batch(batch, as_arrays=True)
    assert mins.shape == (count, n) and mins.dtype == np.uint8
    assert [qb.bits_to_int(mins[b]) for b in range(0, count, 97)] == [int(ob[b]) for b in range(0, count, 97)]


@pytest.mark.parametrize("n,k", [(24, 14), (30, 14), (22, 12), (18, 9)])
def test_prefix_eval_hook(n, k):
    c = instances.config_coeffs("D", 2, n=n)
    L = n - k
    count = min(1 << k, 300)
    vals, fields = _lib.prefix_eval(c, k, 0, count)
    sym = np.triu(c, 1) + np.triu(c, 1).T
    for idx in range(0, count, 7):
        x = np.array([(idx << L >> i) & 1 for i in range(n)], dtype=np.float64)
        assert vals[idx] == O.eval_upper(c, x)
        want = np.diag(c)[:L] + sym[:L] @ x
        assert np.array_equal(fields[idx], want), (n, k, idx)


@pytest.mark.parametrize("n", [3, 8, 12, 14])
def test_all_minimizers_tie_heavy(n):
    for rep in range(5):
        c = _tie_heavy(n, 3100 * n + rep, -1, 1)
        inst = qb.QuboInstance(c)
        _, val, mins = O.expected_argmin(c, 0)
        value, bits = qb.all_minimizers(inst)
        got = [qb.bits_to_int(b) for b in bits]
        assert got == [int(x) for x in mins], (n, rep)
        assert value == val
        # parallel tie rule ordering
        m = n // 2
        _, _, mins_m = O.expected_argmin(c, m)
        _, bits_m = qb.all_minimizers(inst, qb.SolveConfig(threads=2, fixed_bits=m, mode="parallel"))
        assert [qb.bits_to_int(b) for b in bits_m] == [int(x) for x in mins_m]


def test_all_minimizers_config_a_and_floats():
    c = instances.config_coeffs("A", 0)
    _, val, mins = O.expected_argmin(c, 0)
    value, bits = qb.all_minimizers(qb.QuboInstance(c))
    assert [qb.bits_to_int(b) for b in bits] == [int(x) for x in mins] and value == val
    z = np.zeros((14, 14))
    value, bits = qb.all_minimizers(qb.QuboInstance(z))
    assert len(bits) == 1 << 14 and qb.bits_to_int(bits[0]) == 0
    c = instances.config_coeffs("B", 1, n=16)
    _, val, mins = O.expected_argmin(c, 0)
    value, bits = qb.all_minimizers(qb.QuboInstance(c))
    assert [qb.bits_to_int(b) for b in bits] == [int(x) for x in mins]


def test_batch_folds_lower_triangle_like_quboinstance():
    rng = np.random.default_rng(11)
    raw = rng.integers(-3, 4, size=(16, 9, 9)).astype(np.float64)  # full (non-triangular) matrices
    mins, vals = qb.solve_batch(raw, as_arrays=True)
    for b in range(16):
        inst = qb.QuboInstance(raw[b])
        sol = qb.solve_incremental(inst)
        assert np.array_equal(mins[b], sol.minimizer) and vals[b] == sol.value
    bad = raw.copy()
    bad[5, 4, 2] = np.inf
    with pytest.raises(ValueError):
        qb.solve_batch(bad)


def test_fieldwalk_variant_matches_table_and_golden(golden):
    """The literal per-step field-walk kernel returns exactly what the table kernel returns."""
    for case in golden["cases"]:
        if case["n"] < 12:
            continue
        c = np.array(case["coeffs"])
        for key, want in case["results"].items():
            if key == "incremental":
                r = _lib.solve(c, variant=_lib.VARIANT_FIELDWALK)
                # chunks with more than 10 free bits use the field walk; smaller ones the table kernel
                assert r.variant == (_lib.VARIANT_FIELDWALK if case["n"] - r.prefix_bits > 10 else _lib.VARIANT_TABLE)
                assert (r.argmin_bits, r.value) == (want["bits"], want["value"]), case["name"]
            elif key.startswith("parallel_m"):
                m = int(key[len("parallel_m"):])
                r = _lib.solve(c, 0, 0, m, variant=_lib.VARIANT_FIELDWALK)
                assert (r.argmin_bits, r.value) == (want["bits"], want["value"]), (case["name"], key)
    for n in (14, 20, 26, 32):
        for name in ("D", "E"):
            c = instances.config_coeffs(name, 5, n=n)
            a = _lib.solve(c)
            b = _lib.solve(c, variant=_lib.VARIANT_FIELDWALK)
            assert (a.argmin_bits, a.value, a.tie_key) == (b.argmin_bits, b.value, b.tie_key), (name, n)
            if n == 32:  # 2^21 chunks of 2^11 states: the field walk runs
                assert b.variant == _lib.VARIANT_FIELDWALK
    c = _tie_heavy(16, 4242)
    a = _lib.solve(c, 0, 0, 5)
    b = _lib.solve(c, 0, 0, 5, variant=_lib.VARIANT_FIELDWALK)
    assert (a.argmin_bits, a.tie_key) == (b.argmin_bits, b.tie_key)


def test_float_path_massive_ties_device_reduction():
    """A non-quantizable (fp64) instance with 2^21 exactly tied minimisers: more than the 2^20
    candidate buffer, so the device re-evaluates every candidate in fp64 and reduces (value, key)."""
    n = 24
    c = np.zeros((n, n))
    rng = np.random.default_rng(5)
    core = np.triu(rng.uniform(-1, 1, size=(3, 3)))
    c[21:, 21:] = core  # bits 0..20 are decoupled with zero cost: every minimum is 2^21-fold tied
    inst = qb.QuboInstance(c)
    res = _lib.solve(inst.coeffs)
    assert res.exact == 0 and res.candidates > (1 << 20)
    bits, val, _ = O.expected_argmin(c, 0)
    assert int(res.argmin_bits) == bits and res.value == val
    for m in (3, 22):
        bits_m, _, _ = O.expected_argmin(c, m)
        r = _lib.solve(inst.coeffs, 0, 0, m)
        assert int(r.argmin_bits) == bits_m, m


@pytest.mark.parametrize("n,m", [(30, 2), (32, 5), (34, 9), (36, 14)])
def test_large_geometry_subspaces_vs_oracle(n, m):
    """Large chunks (outer Gray walk active) with fixed suffix bits: solve_subspace against the
    CPU oracle's exact scan of the same subspace, integer and float instances."""
    rng = np.random.default_rng(n * 100 + m)
    for name in ("D", "E"):
        c = instances.config_coeffs(name, 7, n=n)
        inst = qb.QuboInstance(c)
        for suffix in rng.integers(0, 1 << m, size=2):
            suffix = int(suffix)
            bits, val, ev = O.solve_subspaces(c, m, suffix, suffix + 1)
            sol = qb.solve_subspace(inst, qb.SubspaceSpec(m, suffix))
            assert (_bits(sol), sol.value, sol.evaluations) == (bits, val, ev), (name, n, m, suffix)


def test_large_geometry_parallel_tie_rule_vs_oracle():
    """solve_parallel(m) at n=30 with many exact ties ({-1,0,1} entries): the (suffix, local Gray
    rank) rule on the large-chunk geometry against the reference-order oracle."""
    c = _tie_heavy(30, 777, -1, 1)
    inst = qb.QuboInstance(c)
    for m in (0, 3):
        bits, val, ev = O.solve_subspaces(c, m, threads=16)
        sol = qb.solve_parallel(inst, qb.SolveConfig(threads=8, fixed_bits=m))
        assert (_bits(sol), sol.value, sol.evaluations) == (bits, val, ev), m


def _adversarial(kind, n, seed):
    rng = np.random.default_rng(seed)
    if kind == "big_int":  # |Q| up to 2^30: sums exceed the fp32 exactness bound -> scale-down, filter path
        c = rng.integers(-(1 << 30), 1 << 30, size=(n, n)).astype(np.float64)
    elif kind == "wide_range":  # 1e-10 .. 1e10 magnitudes
        c = rng.standard_normal((n, n)) * 10.0 ** rng.integers(-10, 11, size=(n, n))
    elif kind == "tiny":  # around 1e-300 incl. subnormals
        c = rng.standard_normal((n, n)) * 1e-300
        c[0, 0] = 5e-320
    elif kind == "neg_zero":
        c = rng.integers(-2, 3, size=(n, n)).astype(np.float64)
        c[c == 0] = -0.0
    elif kind == "dyadic":  # exactly representable after scaling: exact path with e > 0
        c = rng.integers(-64, 65, size=(n, n)) / 1024.0
    return np.triu(c)


@pytest.mark.parametrize("kind", ["big_int", "wide_range", "tiny", "neg_zero", "dyadic"])
def test_adversarial_value_ranges_vs_oracle(kind):
    for n in (9, 14, 22):
        for seed in range(3):
            c = _adversarial(kind, n, 1000 * n + seed)
            inst = qb.QuboInstance(c)
            bits, val, ev = O.solve_incremental(inst.coeffs)
            sol = qb.solve_incremental(inst)
            assert (_bits(sol), sol.value) == (bits, val), (kind, n, seed)
            m = 3
            bits, val, _ = O.solve_subspaces(inst.coeffs, m)
            sol = qb.solve_parallel(inst, qb.SolveConfig(threads=2, fixed_bits=m))
            assert (_bits(sol), sol.value) == (bits, val), (kind, n, seed, m)


@pytest.mark.parametrize("n", [31, 33])
def test_coarse_kernel_matches_table_kernel(n):
    """The packed-int16 filter kernel (default for large chunks) returns exactly what the fp32
    table kernel returns: integer and float instances, tie-heavy instances, subspaces, tie rules."""
    cases = [instances.config_coeffs("D", 9, n=n), instances.config_coeffs("E", 9, n=n),
             instances.config_coeffs("B", 9, n=n), _tie_heavy(n, 4100 + n, -1, 1),
             instances.int_uniform_coeffs(n, 4200 + n, -(1 << 20), 1 << 20)]
    for c in cases:
        for args in ((0, 0, 0), (0, 0, 4), (3, 5, 3)):
            a = _lib.solve(c, *args, variant=_lib.VARIANT_TABLE)
            b = _lib.solve(c, *args, variant=_lib.VARIANT_COARSE)
            assert b.variant == _lib.VARIANT_COARSE  # chunks of >= 10 free bits have a coarse kernel
            assert (a.argmin_bits, a.value, a.tie_key) == (b.argmin_bits, b.value, b.tie_key), (n, args)


@pytest.mark.parametrize("kind", ["big_int", "wide_range", "tiny", "neg_zero", "dyadic"])
def test_adversarial_value_ranges_coarse_kernel(kind):
    """The coarse kernel's int16 image (scale shift, bias, certified slack) on adversarial value
    ranges at n=30, against the fp32 table kernel (itself checked against the oracle)."""
    for seed in range(2):
        c = _adversarial(kind, 30, 7000 + seed)
        inst = qb.QuboInstance(c)
        for args in ((0, 0, 0), (0, 0, 5)):
            a = _lib.solve(inst.coeffs, *args, variant=_lib.VARIANT_TABLE)
            b = _lib.solve(inst.coeffs, *args, variant=_lib.VARIANT_COARSE)
            assert b.variant == _lib.VARIANT_COARSE
            assert (a.argmin_bits, a.value, a.tie_key) == (b.argmin_bits, b.value, b.tie_key), (kind, seed, args)


@pytest.mark.parametrize("n", [34, 35])
def test_tc_kernel_matches_table_kernel(n):
    """The tensor-core coarse pass (tcgen05.mma, fp32 TMEM cells holding two states' threshold
    tests) returns exactly what the fp32 table kernel returns: integer, float, tie-heavy and
    wide-range instances, subspaces and tie rules (n >= 34: chunks of >= 14 free bits)."""
    cases = [instances.config_coeffs("D", 9, n=n), instances.config_coeffs("E", 9, n=n),
             instances.config_coeffs("B", 9, n=n), _tie_heavy(n, 4300 + n, -1, 1),
             instances.int_uniform_coeffs(n, 4400 + n, -(1 << 20), 1 << 20)]
    for c in cases:
        for args in ((0, 0, 0), (0, 0, 4), (3, 5, 3)):
            a = _lib.solve(c, *args, variant=_lib.VARIANT_TABLE)
            b = _lib.solve(c, *args, variant=_lib.VARIANT_TC)
            assert b.variant == _lib.VARIANT_TC
            assert (a.argmin_bits, a.value, a.tie_key) == (b.argmin_bits, b.value, b.tie_key), (n, args)


@pytest.mark.parametrize("kind", ["big_int", "wide_range", "tiny", "neg_zero", "dyadic"])
def test_adversarial_value_ranges_tc_kernel(kind):
    """The tensor-core pass's 10-bit coarse image (shift, beta, per-block threshold offset) on
    adversarial value ranges at n=34, against the fp32 table kernel."""
    c = _adversarial(kind, 34, 7100)
    inst = qb.QuboInstance(c)
    for args in ((0, 0, 0), (0, 0, 5)):
        a = _lib.solve(inst.coeffs, *args, variant=_lib.VARIANT_TABLE)
        b = _lib.solve(inst.coeffs, *args, variant=_lib.VARIANT_TC)
        assert b.variant == _lib.VARIANT_TC
        assert (a.argmin_bits, a.value, a.tie_key) == (b.argmin_bits, b.value, b.tie_key), (kind, args)


def test_tc_kernel_sharded_partial_rounds():
    """Shards whose chunk counts are not multiples of the 128-row MMA (inactive rows in the last
    round) combine to the unsharded answer through the tensor-core pass."""
    for name in ("E", "D"):
        c = instances.config_coeffs(name, 3, n=34)
        whole = _lib.solve(c, variant=_lib.VARIANT_TABLE)
        for S in (3, 7):
            parts = [_lib.solve(c, shard=i, shard_count=S, variant=_lib.VARIANT_TC) for i in range(S)]
            assert all(p.variant == _lib.VARIANT_TC for p in parts)
            best = min(parts, key=lambda r: (r.value_key, r.tie_key))
            assert (best.argmin_bits, best.value, best.tie_key) == (whole.argmin_bits, whole.value, whole.tie_key)
            assert sum(p.states for p in parts) == 1 << 34


@pytest.mark.parametrize("name", ["E", "D", "B"])
def test_tc_kernel_n40(name):
    """n=40 through the tensor-core pass (sparse fp32, dense int +-1000, dense fp32): same answer as
    the default coarse kernel."""
    c = instances.config_coeffs(name, 0, n=40)
    a = _lib.solve(c)
    b = _lib.solve(c, variant=_lib.VARIANT_TC)
    assert b.variant == _lib.VARIANT_TC
    assert (a.argmin_bits, a.value, a.tie_key) == (b.argmin_bits, b.value, b.tie_key)


def test_concurrent_host_threads():
    """ctypes releases the GIL: several host threads solving at once (as a thread pool over the
    reference's entry points would) must each get their own correct answer."""
    from concurrent.futures import ThreadPoolExecutor

    cases = [instances.config_coeffs(name, rep, n=n) for name in ("D", "E") for rep in range(4) for n in (18, 26)]
    want = [O.expected_argmin(c, 0)[0] if c.shape[0] <= 20 else None for c in cases]
    serial = [int(_lib.solve(c).argmin_bits) for c in cases]

    def job(i):
        return int(qb.solve_incremental(qb.QuboInstance(cases[i])).minimizer.astype(np.uint64)
                   .dot(np.uint64(1) << np.arange(cases[i].shape[0], dtype=np.uint64)))

    with ThreadPoolExecutor(max_workers=8) as pool:
        got = list(pool.map(job, range(len(cases)) , chunksize=1))
    assert got == serial
    for g, w in zip(got, want):
        if w is not None:
            assert g == w


@pytest.mark.parametrize("name", ["A", "B", "D"])
def test_n40_other_instance_types(name):
    """n=40 with the other BASELINE value distributions (int +-100, dense fp32 N(0,1), int +-1000):
    the default coarse kernel and the fp32 table kernel agree, and the argmin is the exact minimum
    of its own 2^23-state subspace (CPU oracle)."""
    c = instances.config_coeffs(name, 0, n=40)
    a = _lib.solve(c)
    b = _lib.solve(c, variant=_lib.VARIANT_TABLE)
    d = _lib.solve(c, variant=_lib.VARIANT_COARSE)
    assert a.variant in _lib.IMM_VARIANTS
    assert b.variant == _lib.VARIANT_TABLE and d.variant == _lib.VARIANT_COARSE
    assert (a.argmin_bits, a.value, a.tie_key) == (b.argmin_bits, b.value, b.tie_key)
    assert (a.argmin_bits, a.value, a.tie_key) == (d.argmin_bits, d.value, d.tie_key)
    x = int(a.argmin_bits)
    m = 17
    bits, val, _ = O.solve_subspaces(c, m, x >> (40 - m), (x >> (40 - m)) + 1)
    assert bits == x and val == a.value


def test_bench_records_match_reference_bench(bench_golden):
    # the reference's own `qubrute bench` rows (seconds dropped): same instances, same values
    from paper_2310_19373_b200 import benchrec

    a = bench_golden["args"]
    recs = benchrec.run_bench(int(a[2]), int(a[4]), reps=int(a[6]), modes=a[8], threads=int(a[10]))
    assert [(r.n, r.mode, r.rep) for r in recs] == [(n, m, rep) for n, m, rep, _ in bench_golden["rows"]]
    assert [r.value for r in recs] == [float(v) for *_, v in bench_golden["rows"]]
    assert all(r.seconds > 0 for r in recs)
    text = io.StringIO()
    benchrec.write_csv(recs, stream=text)
    assert benchrec.parse_csv(text.getvalue()) == recs


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0]])
def test_batch_across_devices_gathers_in_order(golden, devices):
    """Config C split over a device list (one slice per entry): the gathered answers
    equal the reference's 4096 golden results in order; odd counts and more slices than instances."""
    cb = golden["configC"]
    batch = instances.config_batch(cb["count"], cb["n"])
    bits, vals, _ = _lib.solve_batch_devices(batch, devices)
    assert [int(b) for b in bits] == cb["bits"]
    assert vals.tolist() == cb["values"]
    mins, mvals = qb.solve_batch(batch[:5], as_arrays=True, devices=devices + [0, 0, 0, 0])
    assert [qb.bits_to_int(m) for m in mins] == cb["bits"][:5]
    assert mvals.tolist() == cb["values"][:5]


@pytest.mark.parametrize("n", [12, 14, 16, 17])
def test_batch_warp_kernel_equals_cta_kernel(n, monkeypatch):
    """The warp-per-instance batch kernel (12 <= n <= 17) against the one-CTA-per-instance kernel
    (QB_BATCH_WARP=0) on float, integer and tie-heavy instances, fp32- and fp64-packed inputs."""
    batch = np.stack([instances.normal_coeffs(n, 7000 + b) for b in range(300)]
                     + [instances.int_uniform_coeffs(n, 8000 + b, -3, 3) for b in range(100)]
                     + [_tie_heavy(n, 9000 + b, -1, 1) for b in range(60)])
    batch[333, 1, 2] += 0.1  # one piece ships fp64
    got = _lib.solve_batch(batch)
    monkeypatch.setenv("QB_BATCH_WARP", "0")
    ref = _lib.solve_batch(batch)
    assert [int(b) for b in got[0]] == [int(b) for b in ref[0]]
    assert got[1].tolist() == ref[1].tolist()
