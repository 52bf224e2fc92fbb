"""CPU replay of the byte-packed threshold test (qb_coarse8.cuh) on the image the library builds.

qb_byte_image (host only) returns what the threshold kernels of kind 3..7 (QB_VARIANT_IMM8, IMM8S, IMM8A,
IMM8AS, IMM8AQ) would run an instance with: the packed table words, the quantized instance, fl(1/unit), Rneg and the
certified slack.  This test recomputes, in numpy and with the device's float operations, the bytes
f(z) = base + sum hc_i z_i + Tc8(z) of randomly chosen blocks and checks the two claims the kernel's
correctness rests on:

* range: every byte stays in [1, 255] for every limit (no wrap, no carry between the four bytes of a word);
* no false negatives: whenever a state of the block has an exact (quantized) value <= the pruning threshold,
  the block passes (a byte has bit 7 clear, or the limit is non-negative) -- so pruning never drops a
  minimiser or a tie.
"""

import numpy as np
import pytest

import paper_2310_19373_b200 as qb
from paper_2310_19373_b200 import _lib, instances

B, CB2 = 10, 6


def _decode_words(words):
    """Signed bytes t_j with sum t_j 256^j = word (mod 2^32), the inverse of the host's packing."""
    out = np.zeros(4 * len(words), dtype=np.int64)
    for k, w in enumerate(words):
        v = int(w)
        for j in range(4):
            t = v & 0xFF
            if t >= 128:
                t -= 256
            out[4 * k + j] = t
            v = ((v - t) >> 8) & 0xFFFFFFFF
    return out


def _subset_sums(vals):
    s = np.zeros(1, dtype=np.int64)
    for v in vals:
        s = np.concatenate([s, s + int(v)])
    return s


def _replay(c, kind, rng, nblocks=120):
    words, q, inv, rneg, slack, _e = _lib.byte_image(c, kind)
    n = q.shape[0]
    approx = kind in (5, 6, 7)
    nb = B + {4: 1, 6: 1, 7: 2}.get(kind, 0)
    tc8 = _decode_words(words)
    assert len(tc8) == 1 << nb and np.abs(tc8).max() <= 127
    qs = q + np.triu(q, 1).T  # symmetric, diagonal once
    # exact table over the image bits: T(z) = sum_{i<=j<nb} q_ij z_i z_j
    z = np.arange(1 << nb)
    bits = ((z[:, None] >> np.arange(nb)) & 1).astype(np.float64)
    T = np.einsum("zi,ij,zj->z", bits, np.triu(q)[:nb, :nb], bits).astype(np.int64)
    inv64 = float(inv)
    fails = 0
    for _ in range(nblocks):
        x = rng.integers(0, 2, size=n).astype(np.float64)
        x[:nb] = 0
        V = int(round(x @ np.triu(q) @ x))
        H = np.array([int(round(qs[i, nb:] @ x[nb:])) for i in range(nb)], dtype=np.int64)
        hc = np.rint(H.astype(np.float32) * np.float32(inv)).astype(np.int64)  # FMUL + F2I (round to nearest even)
        exact = V + _subset_sums(H) + T
        lin = _subset_sums(hc[:CB2])  # w part
        rows = _subset_sums(hc[CB2:nb])
        amin = int(np.minimum(hc[CB2:nb], 0).sum())
        row_term = np.full_like(rows, amin) if approx else rows
        coarse = (row_term[:, None] + lin[None, :]).reshape(-1) + tc8  # z = (u << 6) | w
        bmin = int(exact.min())
        for thr in (bmin, bmin - 1, bmin + 1, bmin + slack, bmin - slack, bmin + 7 * slack, int(exact.max()),
                    bmin + int(rng.integers(-3 * slack - 3, 3 * slack + 3))):
            d = thr + slack - V
            lrel = int(np.floor(np.float32(float(np.float32(d)) * inv64 + 2.0 ** -10)))
            lc = min(max(lrel, -rneg - 1), -1)
            f = 127 - lc + coarse
            assert f.min() >= 1 and f.max() <= 255, (kind, f.min(), f.max(), rneg)
            passed = lrel >= 0 or bool((f < 128).any())
            if (exact <= thr).any() and not passed:
                fails += 1
    return fails


CASES = [("E", 40, 0), ("E", 33, 3), ("D", 32, 0), ("D", 36, 1), ("B", 34, 2), ("A", 36, 5)]


@pytest.mark.parametrize("kind", [3, 4, 5, 6, 7])
@pytest.mark.parametrize("name,n,rep", CASES)
def test_byte_image_range_and_no_false_negatives(name, n, rep, kind):
    c = instances.config_coeffs(name, rep, n=n)
    assert _replay(c, kind, np.random.default_rng(1000 * kind + n)) == 0


@pytest.mark.parametrize("kind", [3, 4, 5, 6, 7])
def test_byte_image_tie_heavy_and_wide_range(kind):
    rng = np.random.default_rng(kind)
    assert _replay(instances.int_uniform_coeffs(33, 777, -1, 1), kind, rng) == 0
    n = 32
    c = np.zeros((n, n))
    c[0, 0] = -1.0e9
    iu = np.triu_indices(n, 1)
    c[iu] = np.random.default_rng(5).standard_normal(len(iu[0])) * 1e-3
    assert _replay(qb.QuboInstance(c).coeffs, kind, rng, nblocks=40) == 0
    assert _replay(np.zeros((n, n)), kind, rng, nblocks=5) == 0
