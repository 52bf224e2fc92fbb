"""Development timing helper: per-config kernel / call times of the GPU solve."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2310_19373_b200 import _lib, instances

out = {}
for name in sys.argv[1:] or ["A", "B", "D", "E"]:
    c = instances.config_coeffs(name, 0)
    n = c.shape[0]
    for _ in range(2):
        r = _lib.solve(c)
    ks, ts, ss = [], [], []
    for _ in range(5):
        t0 = time.perf_counter()
        r = _lib.solve(c)
        ts.append((time.perf_counter() - t0) * 1e3)
        ks.append(r.kernel_ms)
        ss.append(r.search_ms)
    km, tm, sm = float(np.median(ks)), float(np.median(ts)), float(np.median(ss))
    out[name] = dict(n=n, kernel_ms=km, search_ms=sm, search_min=min(ss), search_max=max(ss), call_ms=tm, states_per_s_kernel=2**n / (km * 1e-3),
                     states_per_s_call=2**n / (tm * 1e-3), exact=r.exact, k=r.prefix_bits, e=r.scale_exp,
                     cand=r.candidates, value=r.value, argmin=hex(r.argmin_bits))
    import subprocess
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    out[name]["smi_after"] = clk
    print(name, json.dumps(out[name]), flush=True)
