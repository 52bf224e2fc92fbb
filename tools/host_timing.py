"""Development helper: run small solves against a QB_HOST_TIMING build and average the phase marks."""
import collections, os, subprocess, sys
lib = sys.argv[1]
code = r'''
import sys; sys.path.insert(0, ".")
from paper_2310_19373_b200 import _lib, instances
for name in %r:
    c = instances.config_coeffs(name, 0)
    for _ in range(50): _lib.solve(c)
    print("=== " + name, file=sys.stderr, flush=True)
    for _ in range(100): _lib.solve(c)
''' % (sys.argv[2:] or ["A", "B"],)
p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, QB_LIB_PATH=lib), capture_output=True, text=True)
cur = None
acc = collections.defaultdict(lambda: collections.defaultdict(list))
for ln in p.stderr.splitlines():
    if ln.startswith("=== "):
        cur = ln[4:]
    elif ln.startswith("qbt ") and cur:
        _, tag, v = ln.split()
        acc[cur][tag].append(float(v))
for name, tags in acc.items():
    print(name, " ".join(f"{t}={sorted(v)[len(v) // 2]:.1f}" for t, v in tags.items()))
