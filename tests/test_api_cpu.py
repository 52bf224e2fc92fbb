"""Host-side API contract (no GPU): validation and error types mirror the reference
(solver.py / core.py), raised before any device work."""

import numpy as np
import pytest

import paper_2310_19373_b200 as qb


def test_instance_validation():
    with pytest.raises(ValueError, match="square"):
        qb.QuboInstance(np.zeros((2, 3)))
    with pytest.raises(ValueError, match="at least 1"):
        qb.QuboInstance(np.zeros((0, 0)))
    with pytest.raises(qb.DimensionCapError, match="cap"):
        qb.QuboInstance(np.zeros((41, 41)))
    with pytest.raises(ValueError, match="finite"):
        qb.QuboInstance([[np.nan]])
    with pytest.raises(ValueError, match="strict"):
        qb.QuboInstance([[0.0, 0.0], [1.0, 0.0]], strict=True)
    inst = qb.QuboInstance([[1.0, 2.0], [3.0, 4.0]])
    assert inst.coeffs.tolist() == [[1.0, 5.0], [0.0, 4.0]]
    assert not inst.coeffs.flags.writeable


def test_solver_validation_before_device_work():
    inst = qb.random_instance(6, seed=1)
    with pytest.raises(ValueError):
        qb.SolveConfig(threads=0)
    with pytest.raises(ValueError):
        qb.SolveConfig(mode="annealing")
    with pytest.raises(ValueError):
        qb.solve_parallel(inst, qb.SolveConfig(fixed_bits=6))
    with pytest.raises(ValueError):
        qb.solve_parallel(qb.random_instance(1, seed=1))
    with pytest.raises(ValueError):
        qb.SubspaceSpec(m=2, suffix=4)
    with pytest.raises(ValueError):
        qb.SubspaceSpec(m=-1, suffix=0)
    with pytest.raises(ValueError):
        qb.solve_subspace(qb.random_instance(4, seed=1), qb.SubspaceSpec(m=4, suffix=0))
    with pytest.raises(qb.DimensionCapError, match="guard"):
        qb.solve_naive(qb.random_instance(10, seed=1), max_n=8)
    with pytest.raises(qb.DimensionCapError):
        qb.solve_incremental(qb.QuboInstance(np.zeros((41, 41)), max_n=41))


def test_default_fixed_bits_and_combine():
    assert [qb.default_fixed_bits(10, t) for t in (1, 2, 3, 8)] == [0, 1, 2, 3]
    assert qb.default_fixed_bits(3, 16) == 2
    sols = [qb.Solution(np.array([s], dtype=np.uint8), v, 1, 1e-9) for s, v in enumerate([0.0, -2.3, -1.8, 0.2])]
    assert qb.combine_subspace_minima(sols).value == -2.3
    ties = [qb.Solution(np.array([s], dtype=np.uint8), -1.0, 1, 1e-9) for s in range(3)]
    assert qb.combine_subspace_minima(ties).minimizer[0] == 0
    with pytest.raises(ValueError):
        qb.combine_subspace_minima([])


def test_gray_helpers():
    assert [qb.ctz(k) for k in range(1, 9)] == [0, 1, 0, 2, 0, 1, 0, 3]
    for w in range(1, 12):
        perm = qb.gray_permutation(w)
        assert sorted(perm) == list(range(1 << w))
        assert all(qb.gray_rank(g) == t for t, g in enumerate(perm))
    assert list(qb.flip_sequence(3)) == [0, 1, 0, 2, 0, 1, 0]


def test_delta_and_split_consistency():
    inst = qb.random_instance(9, seed=5)
    form = qb.split(inst)
    x = np.zeros(9, dtype=np.uint8)
    v = 0.0
    for l in qb.flip_sequence(9):
        x[l] ^= 1
        v += qb.delta(form, x, l)
        assert abs(v - qb.evaluate(inst, x)) <= 1e-9


def test_solve_config_devices_validation():
    # extension knob: devices to shard over, validated like the reference's knobs
    assert qb.SolveConfig(devices=[0, 1]).devices == (0, 1)
    assert qb.SolveConfig().devices is None
    for bad in ([], [-1], ["0"]):
        with pytest.raises(ValueError):
            qb.SolveConfig(devices=bad)


def test_step_level_drift_pinned_to_reference(golden):
    """Acceptance criterion 2 shape (reference test_acceptance.py:56-73): the running value after each
    Eq. 3 ``delta`` along the Gray walk, bit-identical to the reference's own trace (every 97th step
    of the n=12 walk, tests/golden/reference_golden.json ``delta_trace_n12``), and within 1e-9 of the
    direct evaluation at every step."""
    tr = golden["delta_trace_n12"]
    inst = qb.QuboInstance(np.array(tr["coeffs"]))
    form = qb.split(inst)
    want = {k: (l, v, d) for k, l, v, d in tr["samples"]}
    x = np.zeros(12, dtype=np.uint8)
    v = 0.0
    seen = 0
    for k, l in enumerate(qb.flip_sequence(12), start=1):
        x[l] ^= 1
        v += qb.delta(form, x, l)
        if k in want:
            wl, wv, wd = want[k]
            assert (l, v) == (wl, wv), k
            assert qb.evaluate(inst, x) == wd
            seen += 1
        assert abs(v - qb.evaluate(inst, x)) <= 1e-9
    assert seen == len(want) > 40


def test_step_level_drift_full_traces():
    """The same pin at every one of the 4095 steps, for two instances (make_golden_extra.py)."""
    import json
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", "reference_golden_extra.json")
    with open(path) as fh:
        traces = json.load(fh)["drift_traces"]
    for tr in traces:
        inst = qb.random_instance(tr["n"], tr["seed"])
        form = qb.split(inst)
        x = np.zeros(tr["n"], dtype=np.uint8)
        v = 0.0
        for k, l in enumerate(qb.flip_sequence(tr["n"])):
            x[l] ^= 1
            v += qb.delta(form, x, l)
            assert l == tr["flips"][k]
            assert v == float.fromhex(tr["running_hex"][k]), k
            assert qb.evaluate(inst, x) == float.fromhex(tr["direct_hex"][k]), k
