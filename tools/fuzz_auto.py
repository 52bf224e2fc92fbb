"""Randomised parity soak of the byte-packed kernels and AUTO's policy against the table-load kernels.

python tools/fuzz_auto.py [cases] [seed]: random instance families, sizes n = 31..37, optional fixed bits, tie
parameter and shards; every variant and two AUTO solves must return the table-load coarse kernel's answer (for
shards: the combined answer)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib, instances

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)


def make(n):
    iu = np.triu_indices(n, 1)
    m = len(iu[0])
    fam = int(rng.integers(0, 9))
    c = np.zeros((n, n))
    if fam == 0:    # sparse normal
        dens = rng.choice([0.02, 0.1, 0.3])
        c[iu] = rng.standard_normal(m) * (rng.random(m) < dens); c[np.diag_indices(n)] = rng.standard_normal(n)
    elif fam == 1:  # dense normal (float32-valued)
        c[iu] = rng.standard_normal(m).astype(np.float32); c[np.diag_indices(n)] = rng.standard_normal(n).astype(np.float32)
    elif fam == 2:  # dense integers, random scale
        s = int(rng.choice([1, 3, 100, 1000, 30000]))
        c[iu] = rng.integers(-s, s + 1, m); c[np.diag_indices(n)] = rng.integers(-s, s + 1, n)
    elif fam == 3:  # tie-heavy
        c[iu] = rng.integers(-1, 2, m); c[np.diag_indices(n)] = rng.integers(-1, 2, n)
    elif fam == 4:  # antiferromagnetic
        c[iu] = rng.random(m); c[np.diag_indices(n)] = -rng.random(n) * rng.choice([2, 8, 16])
    elif fam == 5:  # ferromagnetic
        c[iu] = -rng.random(m); c[np.diag_indices(n)] = rng.random(n) * 3
    elif fam == 6:  # wide range
        c[iu] = rng.standard_normal(m) * np.where(rng.random(m) < 0.05, 1e3, 1e-3); c[np.diag_indices(n)] = rng.standard_normal(n)
    elif fam == 7:  # one huge term
        c[iu] = rng.standard_normal(m) * 1e-3; c[0, 0] = -1e9 * rng.random()
    else:           # mostly zero
        k = rng.integers(0, m, 5); c[iu[0][k], iu[1][k]] = rng.standard_normal(5)
    return fam, c


def key(r):
    return (int(r.value_key), int(r.tie_key))


bad = 0
t0 = time.time()
for t in range(cases):
    n = int(rng.integers(31, 38))
    fam, c = make(n)
    m_fix = int(rng.choice([0, 0, 0, 2, 5]))
    suffix = int(rng.integers(0, 1 << m_fix)) if m_fix else 0
    m_tie = m_fix + int(rng.choice([0, 0, 3, 7]))
    shards = int(rng.choice([1, 1, 1, 2, 3]))
    def run(var):
        rs = [_lib.solve(c, m_fix, suffix, m_tie, shard=s, shard_count=shards, variant=var) for s in range(shards)]
        return min(rs, key=key)
    t1 = time.time()
    ref = run(_lib.VARIANT_COARSE)
    if time.time() - t1 > 2.0:
        print(f"SLOW case {t} fam {fam} n {n} COARSE: {time.time() - t1:.1f} s kernel_ms {ref.kernel_ms:.1f} search {ref.search_ms:.1f} collect {ref.collect_ms:.1f} cand {ref.candidates}", flush=True)
    want = (int(ref.argmin_bits), ref.value, int(ref.tie_key))
    got = {}
    for var in (_lib.VARIANT_BYTE8, _lib.VARIANT_IMM8, _lib.VARIANT_IMM8S, _lib.VARIANT_IMM8A, _lib.VARIANT_IMM8AS,
                _lib.VARIANT_IMM8AQ, _lib.VARIANT_AUTO, _lib.VARIANT_AUTO, _lib.VARIANT_AUTO):
        t1 = time.time()
        r = run(var)
        if time.time() - t1 > 2.0:
            print(f"SLOW case {t} fam {fam} n {n} m_fix {m_fix} m_tie {m_tie} shards {shards} var {var} used {r.variant}: {time.time() - t1:.1f} s "
                  f"kernel_ms {r.kernel_ms:.1f} search_ms {r.search_ms:.1f} collect_ms {r.collect_ms:.1f} cand {r.candidates} exact_blocks {r.exact_blocks} exact {r.exact}", flush=True)
        got[var] = (int(r.argmin_bits), r.value, int(r.tie_key))
        if got[var] != want:
            bad += 1
            print(f"MISMATCH case {t} fam {fam} n {n} m_fix {m_fix} m_tie {m_tie} shards {shards} var {var} -> used {r.variant}: "
                  f"{got[var]} != {want}", flush=True)
    if t % 10 == 0:
        print(f"case {t}: fam {fam} n {n} m_fix {m_fix} m_tie {m_tie} shards {shards} ok ({time.time() - t0:.0f} s)", flush=True)
print(f"fuzz done: {cases} cases, {bad} mismatches")
