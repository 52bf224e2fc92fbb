"""GPU parity of the patched-immediate coarse kernels (QB_VARIANT_IMM: 10-bit blocks; QB_VARIANT_IMM2:
11-bit super-blocks, AUTO's default where the coarse filter runs): the instance's coarse table is
written into the kernel's SASS as instruction immediates (qb_api.cu imm_kernel / imm_patch).  Every
result must equal the table-load coarse kernel's (same blocks, same certified bounds, same tie keys)
and, where affordable, the oracle's."""

import numpy as np
import pytest

import paper_2310_19373_b200 as qb
from oracle import oracle as O
from paper_2310_19373_b200 import _lib, instances

pytestmark = pytest.mark.gpu


def _same(a, b):
    return (int(a.argmin_bits), a.value, int(a.tie_key), int(a.value_key)) == \
        (int(b.argmin_bits), b.value, int(b.tie_key), int(b.value_key))


CASES = [("E", 40, 0), ("E", 40, 1), ("E", 36, 2), ("E", 33, 3), ("D", 32, 0), ("D", 32, 4), ("B", 31, 1),
         ("B", 34, 2), ("A", 32, 5)]


IMMS = list(_lib.IMM_VARIANTS)


@pytest.mark.parametrize("var", IMMS)
@pytest.mark.parametrize("name,n,rep", CASES)
def test_imm_equals_table_load_coarse(name, n, rep, var):
    c = instances.config_coeffs(name, rep, n=n)
    ref = _lib.solve(c, variant=_lib.VARIANT_COARSE)
    got = _lib.solve(c, variant=var)
    assert got.variant in IMMS and ref.variant == _lib.VARIANT_COARSE
    assert _same(got, ref), (name, n, rep)
    auto = _lib.solve(c)  # AUTO: whichever kernel it picks gives the same answer
    assert _same(auto, ref)


@pytest.mark.parametrize("var", IMMS)
@pytest.mark.parametrize("m_fix,m_tie,shards", [(0, 6, 1), (0, 0, 3), (4, 4, 1), (2, 9, 2)])
def test_imm_subspaces_ties_and_shards(m_fix, m_tie, shards, var):
    """Tie-heavy integer instance (values in {-1,0,1}): subspace solves, the parallel tie rule and
    shards all agree between the two coarse kernels."""
    c = instances.int_uniform_coeffs(33, 777, -1, 1)
    suffix = 3 if m_fix else 0
    refs = [_lib.solve(c, m_fix, suffix, m_tie, shard=sh, shard_count=shards, variant=_lib.VARIANT_COARSE)
            for sh in range(shards)]
    gots = [_lib.solve(c, m_fix, suffix, m_tie, shard=sh, shard_count=shards, variant=var) for sh in range(shards)]
    key = lambda r: (int(r.value_key), int(r.tie_key))  # noqa: E731 - the combine's order (lower wins)
    win = min(refs, key=key)
    assert _same(min(gots, key=key), win), (m_fix, m_tie)
    for sh, (got, ref) in enumerate(zip(gots, refs)):
        # shards start from the host seed, a value attained somewhere in the searched space: a shard with no
        # state at or below it may come back empty (keys ~0) or with some attained value above it -- never
        # better than its true minimum, and only ever a shard that does not hold the answer (the combine's
        # result above is what the reference defines)
        if not _same(got, ref):
            assert shards > 1 and key(ref) > key(win), (m_fix, m_tie, sh)
            assert int(got.value_key) >= int(ref.value_key), (m_fix, m_tie, sh)


@pytest.mark.parametrize("var", IMMS)
def test_imm_module_cache_alternating_instances(var):
    """More distinct instances than the per-device module cache holds (4), solved twice in
    alternating order: every answer is the one of its own instance (cache keyed by table + L)."""
    cs = [instances.config_coeffs("E", 10 + r, n=32) for r in range(6)]
    want = [_lib.solve(c, variant=_lib.VARIANT_COARSE) for c in cs]
    for _ in range(2):
        for c, w in zip(cs, want):
            assert _same(_lib.solve(c, variant=var), w)


@pytest.mark.parametrize("var", IMMS)
def test_imm_vs_oracle_subspace_n34(var):
    """Oracle check of an IMM search on a float instance: solve_subspace over 2^26 states."""
    c = instances.config_coeffs("E", 7, n=34)
    m, suffix = 8, 77
    got = _lib.solve(c, m, suffix, m, variant=var)
    # (the table-load byte kernel exists for chunks of >= 12 free bits; this geometry has shorter ones and
    # QB_VARIANT_BYTE8 then runs the 16-bit table-load kernel)
    assert got.variant in IMMS or (var == _lib.VARIANT_BYTE8 and got.variant == _lib.VARIANT_COARSE)
    bits, val, _ = O.solve_subspaces(c, m, suffix, suffix + 1, threads=8)
    assert int(got.argmin_bits) == bits and got.value == val


def test_auto_policy_first_solve_and_repeat():
    """AUTO takes a patched kernel on a first solve only when the search is long (n=40), and on
    the repeat of an instance it has seen (n=33); a first n=33 solve runs a table-load kernel (the byte
    kernel, no module to load)."""
    c33 = instances.config_coeffs("E", 41, n=33)
    first = _lib.solve(c33)
    again = _lib.solve(c33)
    assert first.variant == _lib.VARIANT_BYTE8 and int(first.module_ms * 1e6) == 0
    assert again.variant in IMMS and again.variant != _lib.VARIANT_BYTE8
    assert _same(first, again)
    c40 = instances.config_coeffs("E", 42, n=40)
    assert _lib.solve(c40).variant in IMMS


@pytest.mark.parametrize("var", IMMS)
def test_imm_adversarial_ranges(var):
    """Wide-range weights (one huge term, many tiny non-integer ones) and an all-zero instance."""
    n = 32
    c = np.zeros((n, n))
    c[0, 0] = -1.0e9
    rng = np.random.default_rng(5)
    iu = np.triu_indices(n, 1)
    c[iu] = rng.standard_normal(len(iu[0])) * 1e-3
    inst = qb.QuboInstance(c)
    ref = _lib.solve(inst.coeffs, variant=_lib.VARIANT_COARSE)
    got = _lib.solve(inst.coeffs, variant=var)
    assert _same(got, ref)
    z = np.zeros((n, n))
    assert _same(_lib.solve(z, variant=var), _lib.solve(z, variant=_lib.VARIANT_COARSE))


def test_imm2_tie_heavy_against_oracle_full():
    """Super-blocks on a tie-heavy integer instance (values in {-1,0,1}) at n=31: the kernel's
    half-block keys j = 2 j' + (b ^ (j' & 1)) must reproduce the reference's global Gray-rank tie
    rule; checked against the oracle's full solve and solve_parallel(m=5)."""
    c = instances.int_uniform_coeffs(31, 31337, -1, 1)
    for m_tie in (0, 5):
        got = _lib.solve(c, 0, 0, m_tie, variant=_lib.VARIANT_IMM2)
        assert got.variant == _lib.VARIANT_IMM2, got.prefix_bits
        if m_tie == 0:
            bits, val, _ = O.solve_incremental(c)
        else:
            bits, val, _ = O.solve_subspaces(c, m_tie, threads=8)
        assert int(got.argmin_bits) == bits and got.value == val


@pytest.mark.parametrize("scale", [1.0, 0.37])
def test_auto_gives_up_on_a_dense_instance_and_retries(scale):
    """AUTO's optimistic run: on dense integers in +-1000 at n=36 the row-bound byte kernels re-evaluate far
    more than 1 block in 2^10, so the run gives up and the solve is repeated with a tighter kernel
    (qb_result.retries); the answer is the table-load kernel's either way, on the exact path (scale 1) and on
    the certified collect path (non-integer coefficients, scale 0.37)."""
    c = instances.config_coeffs("D", 0, n=36) * scale
    ref = _lib.solve(c, variant=_lib.VARIANT_COARSE)
    first = _lib.solve(c)            # first solve of a short instance: a table-load kernel (the byte kernel gives up)
    runs = [_lib.solve(c) for _ in range(3)]
    assert first.variant in (_lib.VARIANT_COARSE, _lib.VARIANT_BYTE8) and int(first.retries) >= 1
    for r in [first] + runs:
        assert _same(r, ref)
    assert all(r.variant in _lib.IMM_VARIANTS for r in runs)
    # the kind that completed is remembered: the last solve starts from it and does not retry
    assert int(runs[-1].retries) == 0 and runs[-1].variant != _lib.VARIANT_IMM8AS
    # an explicit variant never gives up
    forced = _lib.solve(c, variant=_lib.VARIANT_IMM8AS)
    assert forced.variant == _lib.VARIANT_IMM8AS and int(forced.retries) == 0 and _same(forced, ref)
    assert int(forced.exact_blocks) > (2 ** 26 >> 10)


def test_all_minimisers_through_the_byte_kernels(monkeypatch):
    """Every minimiser of a tie-heavy n=32 instance (values in {-1, 0, 1}): the recording search of the
    byte-packed kernels (first solve: table-load form; repeats: patched forms) lists exactly the states the
    16-bit table-load kernel lists (QB_IMM=0), in the same tie order, each with the minimum value."""
    c = instances.int_uniform_coeffs(32, 4242, -1, 1)
    monkeypatch.setenv("QB_IMM", "0")
    v0, xs0, n0 = _lib.all_minimisers(c)
    monkeypatch.delenv("QB_IMM")
    assert n0 >= 1 and len(xs0) == n0
    for _ in range(3):
        v, xs, cnt = _lib.all_minimisers(c)
        assert (v, cnt) == (v0, n0) and np.array_equal(xs, xs0)
    for x in xs0[:8]:
        bits = np.array([(int(x) >> i) & 1 for i in range(32)], dtype=np.float64)
        assert _lib.eval_upper(c, bits) == v0
