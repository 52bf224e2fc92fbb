import sys; sys.path.insert(0,'.')
from paper_2310_19373_b200 import _lib, instances
for name in sys.argv[1:]:
    c = instances.config_coeffs(name, 0)
    for _ in range(3): r = _lib.solve(c)
