"""GPU parity, round 2: the n=40 headline pinned against a full oracle run, full-size B/D cases from
the reference, large ``fixed_bits`` geometries, sharded solves with the host seed, and the collect
pass's list regrowth.  All calls go through the C ABI (libqubrute_b200.so)."""

import json
import os

import numpy as np
import pytest

import paper_2310_19373_b200 as qb
from oracle import oracle as O
from paper_2310_19373_b200 import _lib, instances

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {name}")
    with open(path) as fh:
        return json.load(fh)


def _bits(sol):
    return qb.bits_to_int(sol.minimizer)


def _combine(parts):
    """Lexicographic (value_key, tie_key) minimum over shard results, empty shards (keys ~0) skipped."""
    live = [p for p in parts if p.value_key != (1 << 64) - 1]
    assert live, "every shard came back empty"
    return min(live, key=lambda r: (r.value_key, r.tie_key))


# ------------------------------------------------------------------ config E, n = 40, pinned
@pytest.mark.parametrize("rep", [0, 1])
def test_config_e_n40_pinned_to_full_oracle_run(rep):
    """The headline instance against the oracle's full 2^40-state solve_parallel(m=14) run
    (tests/golden/make_config_e_pin.py): bit-exact argmin and value for solve_incremental,
    solve_parallel(m=6) and solve_parallel(m=14), and for an 8-shard combine (k=22, L=18)."""
    pin = _load("config_e_n40.json").get(f"rep{rep}")
    if pin is None:
        pytest.fail(f"config_e_n40.json has no rep{rep}")
    c = instances.config_coeffs("E", rep)
    assert instances.coeffs_sha256(c) == pin["coeffs_sha256"]
    inst = qb.QuboInstance(c)
    want_bits, want_val = int(pin["argmin"]), float.fromhex(pin["value_hex"])
    inc = qb.solve_incremental(inst)
    assert (_bits(inc), inc.value, inc.evaluations) == (want_bits, want_val, (1 << 40) - 1)
    for m in (6, 14):
        par = qb.solve_parallel(inst, qb.SolveConfig(threads=8, fixed_bits=m))
        assert (_bits(par), par.value, par.evaluations) == (want_bits, want_val, (1 << 40) - (1 << m)), m
    parts = [_lib.solve(inst.coeffs, shard=i, shard_count=8) for i in range(8)]
    best = _combine(parts)
    assert (int(best.argmin_bits), best.value) == (want_bits, want_val)
    assert sum(p.states for p in parts) == 1 << 40


# ------------------------------------------------------------------ full-size reference cases
def test_reference_full_size_extra_cases():
    """Config B (n=24) reps 1-2 and config D (n=32) incremental / parallel(m=6), as the reference
    solved them (tests/golden/make_golden_extra.py)."""
    g = _load("reference_golden_extra.json")
    for case in g["cases"]:
        c = instances.config_coeffs(case["config"], case["rep"])
        assert instances.coeffs_sha256(c) == case["sha256"]
        inst = qb.QuboInstance(c)
        for key, want in case["results"].items():
            if key == "incremental":
                sol = qb.solve_incremental(inst)
            else:
                m = int(key[len("parallel_m"):])
                sol = qb.solve_parallel(inst, qb.SolveConfig(threads=8, fixed_bits=m))
            got = (_bits(sol), sol.value, sol.evaluations)
            assert got == (want["bits"], want["value"], want["evaluations"]), (case["config"], case["rep"], key)


# ------------------------------------------------------------------ geometry: large fixed_bits
@pytest.mark.parametrize("m", [9, 12, 16, 20])
def test_parallel_large_fixed_bits_n40(m):
    """solve_parallel at n=40 with many fixed bits (threads=512 -> m=9 by default): the chunk count
    follows the searched states, not 2^(m + 19), and the answer equals the m=0 solve
    (the config E minimum is unique, so every tie rule picks it)."""
    c = instances.config_coeffs("E", 0)
    inst = qb.QuboInstance(c)
    ref = qb.solve_incremental(inst)
    r = _lib.solve(inst.coeffs, 0, 0, m)
    assert r.prefix_bits <= max(m, 22)
    sol = qb.solve_parallel(inst, qb.SolveConfig(threads=1 << m))
    assert (_bits(sol), sol.value, sol.evaluations) == (_bits(ref), ref.value, (1 << 40) - (1 << m))


def test_parallel_large_fixed_bits_tie_rule_n32():
    """Tie-heavy integer instance at n=32 with fixed_bits=12: the (suffix, local Gray rank) rule still
    holds when the chunk prefix is driven by m_tie; checked against the oracle's full solve_parallel."""
    c = instances.int_uniform_coeffs(32, 4242, -1, 1)
    inst = qb.QuboInstance(c)
    m = 12
    sol = qb.solve_parallel(inst, qb.SolveConfig(threads=1, fixed_bits=m))
    bits, val, ev = O.solve_subspaces(c, m, threads=os.cpu_count() or 8)
    assert (_bits(sol), sol.value, sol.evaluations) == (bits, val, ev)


# ------------------------------------------------------------------ sharding with the host seed
@pytest.mark.parametrize("name,n,S", [("E", 40, 8), ("D", 32, 8), ("D", 32, 3), ("E", 36, 5), ("B", 34, 4)])
def test_sharded_solves_use_seed_and_combine(name, n, S):
    """Shards now start from the global host seed; a shard whose blocks are all certified above it
    comes back empty (keys ~0) and the (value_key, tie_key) combine equals the one-launch answer."""
    c = instances.config_coeffs(name, 3, n=n)
    whole = _lib.solve(c)
    for m_tie in (0, 5):
        whole = _lib.solve(c, 0, 0, m_tie)
        parts = [_lib.solve(c, 0, 0, m_tie, shard=i, shard_count=S) for i in range(S)]
        best = _combine(parts)
        assert (best.argmin_bits, best.value, best.tie_key) == (whole.argmin_bits, whole.value, whole.tie_key)
        assert sum(p.states for p in parts) == 1 << n
        r = _lib.solve_devices(c, [0] * S, 0, 0, m_tie)
        assert (r.argmin_bits, r.value, r.tie_key) == (whole.argmin_bits, whole.value, whole.tie_key)


# ------------------------------------------------------------------ collect-list regrowth
def test_collect_lists_regrow_on_overflow():
    """One huge diagonal weight and small non-integer weights that quantize to 0: every state with
    x0 = 1 ties in the quantized image, so 2^21 blocks (> the 2^20-entry lists) and 2^31 states fall
    inside the certified bound.  The lists grow and the collect pass reruns; the 2^31 candidates are
    reduced on the device in fp64.  The exact answer is known in closed form."""
    n = 32
    c = np.zeros((n, n))
    c[0, 0] = -1.0e12
    rng = np.random.default_rng(11)
    small = rng.uniform(0.25, 1.0, size=n - 1) * 1e-3
    sign = np.where(np.arange(1, n) % 3 == 0, -1.0, 1.0)
    for i in range(1, n):
        c[i, i] = sign[i - 1] * small[i - 1]
    inst = qb.QuboInstance(c)
    want = 1 | sum(1 << i for i in range(1, n) if c[i, i] < 0)
    r = _lib.solve(inst.coeffs)
    assert r.exact == 0 and r.candidates > (1 << 20)
    assert int(r.argmin_bits) == want
    assert r.value == O.eval_upper(inst.coeffs, qb.bits_from_int(want, n).astype(np.float64))
    sol = qb.solve_incremental(inst)
    assert _bits(sol) == want


# ------------------------------------------------------------------ single-process NCCL combine
def test_solve_devices_nccl_combine(monkeypatch):
    """qb_solve_devices combines shards with one ncclAllReduce(MIN) when its devices are distinct
    (QB_NCCL=1 takes that path for the single GPU here, a one-rank communicator); the answer equals
    the one-launch solve.  With a repeated device the host combine runs (combine == 0)."""
    c = instances.config_coeffs("D", 5, n=30)
    whole = _lib.solve(c)
    monkeypatch.setenv("QB_NCCL", "1")
    r = _lib.solve_devices(c, [0])
    assert r.combine == 1
    assert (r.argmin_bits, r.value, r.tie_key) == (whole.argmin_bits, whole.value, whole.tie_key)
    r2 = _lib.solve_devices(c, [0, 0])
    assert r2.combine == 0
    assert (r2.argmin_bits, r2.value, r2.tie_key) == (whole.argmin_bits, whole.value, whole.tie_key)


@pytest.mark.gpu
def test_solve_batch_float32_input_matches_fp64():
    """A float32 (count, n, n) batch goes to qb_solve_batch_f32 without an fp64 copy; results are those of the
    same batch converted to fp64 (config C: fp32-valued U[-1, 1) entries), including a lower-triangular
    entry that the native fold adds into the upper triangle."""
    import paper_2310_19373_b200 as qb
    from paper_2310_19373_b200 import instances

    b64 = instances.config_batch(300, 16)
    b32 = b64.astype(np.float32)
    assert np.array_equal(b32.astype(np.float64), b64)  # config C values are float32-representable
    b32[7, 5, 2] = np.float32(0.3)  # below the diagonal: folded into (2, 5)
    b64 = b32.astype(np.float64)
    m32, v32 = qb.solve_batch(b32, as_arrays=True)
    m64, v64 = qb.solve_batch(b64, as_arrays=True)
    assert np.array_equal(m32, m64) and np.array_equal(v32, v64)
    sol = qb.solve_incremental(qb.QuboInstance(b64[7]))
    assert np.array_equal(m32[7], sol.minimizer) and v32[7] == sol.value
    bad = b32.copy()
    bad[3, 1, 1] = np.inf
    with pytest.raises(ValueError, match="finite"):
        qb.solve_batch(bad, as_arrays=True)


# ------------------------------------------------------------------ the reference's drift-decided ties
def test_first_minimiser_in_gray_order_where_the_reference_drifts():
    """Float instances with exact ties (free variables) or a huge coefficient: the reference keeps the state whose
    RUNNING value is lowest, and rounding drift of that value decides between exactly tied states (16 of the 99
    reference answers in tests/golden/reference_drift_cases.json; the oracle reproduces them, tests/test_oracle.py).
    This library returns the stated contract instead ("first minimizer in GRAY order"): the lowest
    evaluate() value and, among equal values, the lowest (suffix, Gray rank) key -- found by full enumeration with
    the reference's own evaluate() when the fixture was made.  The value always equals the reference's."""
    fx = _load("reference_drift_cases.json")
    differ = 0
    for case in fx["cases"]:
        c = np.array(case["coeffs"], dtype=np.float64)
        for m, want in case["results"].items():
            for var in (_lib.VARIANT_AUTO, _lib.VARIANT_TABLE, _lib.VARIANT_COARSE, _lib.VARIANT_IMM8AS):
                r = _lib.solve(c, 0, 0, int(m), variant=var)
                assert (int(r.argmin_bits), r.value) == (want["contract_bits"], want["contract_value"]), \
                    (case["kind"], case["n"], m, var)
                assert r.value == want["reference_value"]
            differ += want["contract_bits"] != want["reference_bits"]
        # the package entry points (Seam 2) return the same state
        inst = qb.QuboInstance(c)
        sol = qb.solve_incremental(inst)
        assert (_bits(sol), sol.value) == (case["results"]["0"]["contract_bits"], case["results"]["0"]["contract_value"])
        sol = qb.solve_parallel(inst, qb.SolveConfig(threads=4, fixed_bits=2))
        assert (_bits(sol), sol.value) == (case["results"]["2"]["contract_bits"], case["results"]["2"]["contract_value"])
    assert differ == fx["drift_decided_results"]


# ------------------------------------------------------------------ randomised soaks against the oracle (short forms)
@pytest.mark.parametrize("tool,args", [("fuzz_oracle.py", ["40", "5", "12", "22"]), ("fuzz_batch.py", ["8", "11"])])
def test_randomised_soak_against_oracle_and_enumeration(tool, args):
    """Short runs of tools/fuzz_oracle.py (every kernel variant and AUTO against the oracle and, for n <= 20, a full
    enumeration of evaluate()) and tools/fuzz_batch.py (batch kernels, float32 input, all-minimisers).  The long runs
    are recorded in profiles/r14_fuzz_*.log.  Exit status 1 = an answer the GPU should not have returned."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    run = subprocess.run([sys.executable, os.path.join(root, "tools", tool), *args], capture_output=True, text=True,
                         timeout=900)
    assert run.returncode == 0, run.stdout[-3000:] + run.stderr[-3000:]
    assert "0 mismatches (BUG)" in run.stdout
