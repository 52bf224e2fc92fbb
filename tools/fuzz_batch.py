"""Randomised parity soak of the batch kernels (qb_solve_batch: warp-per-instance for 12 <= n <= 17, CTA-per-instance
otherwise, float32 and fp64 input) and of qb_all_minimisers, on the instance families of tools/fuzz_common.py.

python tools/fuzz_batch.py [rounds] [seed]: each round draws n in 2..20 and a batch of 24..96 instances of mixed
families.  Every instance's answer is compared with
  * a full enumeration of evaluate() in the reference's order (this library's contract: lowest value, then lowest Gray
    rank) -- any difference is a BUG;
  * the oracle's solve_incremental restatement -- a difference there must classify as reference-drift (fuzz_oracle.py).
The same batch also goes through the single-instance path, as a float32 array when it is fp32-representable, and the
first instances of each round through qb_all_minimisers (the complete tie set, sorted by Gray rank)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker, never the product path)
from fuzz_common import make, classify, truth, gray_rank  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 4096)
bad = drift = inst_total = allmin_total = 0
t0 = time.time()
for t in range(rounds):
    n = int(rng.integers(2, 21))
    count = int(rng.integers(24, 97))
    fams, cs = zip(*[make(rng, n) for _ in range(count)])
    if t % 3 == 0:  # every third round: the same instances rounded to float32 values, so the float32 entry point runs
        cs = tuple(c.astype(np.float32).astype(np.float64) for c in cs)
    batch = np.stack(cs)
    bits, vals, _ = _lib.solve_batch(batch)
    f32ok = bool(np.all(batch.astype(np.float32).astype(np.float64) == batch))
    if f32ok:
        b32, v32, _ = _lib.solve_batch(batch.astype(np.float32))
        if not (np.array_equal(b32, bits) and np.array_equal(v32, vals)):
            bad += 1
            print(f"BUG round {t} n {n}: float32 batch differs from the fp64 batch", flush=True)
    ob, ov = O.solve_batch(batch, threads=os.cpu_count() or 1)[:2]
    for i in range(count):
        own = truth(cs[i], n, 0, None)
        got = (int(bits[i]), float(vals[i]))
        if got != own:
            bad += 1
            print(f"BUG round {t} n {n} instance {i} fam {fams[i]}: batch {got} != enumeration {own}", flush=True)
        if got != (int(ob[i]), float(ov[i])):
            kind = classify(cs[i], n, 0, got[0], int(ob[i]))[0]
            if kind == "BUG":
                bad += 1
                print(f"BUG round {t} n {n} instance {i} fam {fams[i]}: batch {got} != oracle {(int(ob[i]), float(ov[i]))}",
                      flush=True)
            else:
                drift += 1
        if i < 8:
            r = _lib.solve(cs[i])
            if (int(r.argmin_bits), r.value) != own:
                bad += 1
                print(f"BUG round {t} n {n} instance {i} fam {fams[i]}: single solve != enumeration", flush=True)
        if i < 4:
            # the complete tie set: every state whose evaluate() equals the minimum, sorted by Gray rank
            x = np.arange(1 << n, dtype=np.int64)
            v = np.zeros(1 << n)
            for a in range(n):
                xa = ((x >> a) & 1).astype(np.float64)
                for b in range(a, n):
                    if cs[i][a, b] != 0.0:
                        v += cs[i][a, b] * xa * ((x >> b) & 1)
            mins = sorted((int(s) for s in np.nonzero(v == v.min())[0]), key=gray_rank)
            val, states, cnt = _lib.all_minimisers(cs[i], cap=1 << 21)
            allmin_total += 1
            if val != float(v.min()) or cnt != len(mins) or [int(s) for s in states] != mins:
                bad += 1
                print(f"BUG round {t} n {n} instance {i} fam {fams[i]}: all_minimisers count {cnt} value {val!r} != "
                      f"enumeration count {len(mins)} value {float(v.min())!r}", flush=True)
    inst_total += count
    print(f"round {t}: n {n} count {count} float32 {f32ok} ok ({time.time() - t0:.0f} s)", flush=True)
print(f"fuzz_batch done: {rounds} rounds, {inst_total} instances, {allmin_total} all-minimiser sets, {bad} mismatches (BUG), "
      f"{drift} reference answers decided by running-value drift")
sys.exit(1 if bad else 0)
