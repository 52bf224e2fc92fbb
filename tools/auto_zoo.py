"""AUTO against the 16-bit patched kernel on a zoo of instance types (n=38): same answers, times, retries."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib, instances

n = int(sys.argv[1]) if len(sys.argv) > 1 else 38
rng = np.random.default_rng(7)
iu = np.triu_indices(n, 1)

def tri(off, diag):
    c = np.zeros((n, n)); c[iu] = off; c[np.diag_indices(n)] = diag
    return c

zoo = {
    "E sparse 10% N(0,1)": instances.config_coeffs("E", 3, n=n),
    "sparse 2% N(0,1)": tri(rng.standard_normal(len(iu[0])) * (rng.random(len(iu[0])) < 0.02), rng.standard_normal(n)),
    "dense N(0,1)": instances.config_coeffs("B", 3, n=n),
    "dense int +-1000": instances.config_coeffs("D", 3, n=n),
    "maxcut-like int {-1,0,1}": instances.int_uniform_coeffs(n, 99, -1, 1),
    "ferromagnetic (all off-diagonal negative)": tri(-rng.random(len(iu[0])), rng.random(n) * 3),
    "antiferromagnetic (all positive off-diagonal, negative diagonal)": tri(rng.random(len(iu[0])), -rng.random(n) * 8),
    "planted + small noise": tri(rng.standard_normal(len(iu[0])) * 0.05, -np.ones(n)),
    "wide range (1e6 : 1)": tri(rng.standard_normal(len(iu[0])) * np.where(rng.random(len(iu[0])) < 0.05, 1e3, 1e-3),
                               rng.standard_normal(n)),
    "uniform [0,1) dense, diag -n/4": tri(rng.random(len(iu[0])), -np.full(n, n / 4.0)),
}
for name, c in zoo.items():
    ref = _lib.solve(c, variant=_lib.VARIANT_IMM)
    ref = _lib.solve(c, variant=_lib.VARIANT_IMM)
    runs = [_lib.solve(c) for _ in range(4)]
    ok = all((r.argmin_bits, r.value, r.tie_key) == (ref.argmin_bits, ref.value, ref.tie_key) for r in runs)
    print(f"{name:66s} imm {ref.search_ms:7.3f} ms | auto " +
          " ".join(f"v{r.variant}/r{r.retries}/{r.kernel_ms:.3f}" for r in runs) +
          f" | x{runs[-1].exact_blocks} {'OK' if ok else 'MISMATCH'}", flush=True)
