"""Small sweep run for ncu captures: python tools/profile_case.py c4 [cells] [n_mu] [n_az] [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import problem as pb, _capi

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cells = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n_mu = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n_az = int(sys.argv[4]) if len(sys.argv) > 4 else 8
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
P = pb.config(name, cells=cells, n_mu=n_mu, n_az=n_az)
s = pk.SweepSolver(P)
L = _capi.load()
for _ in range(reps):
    assert L.hsw_sweep_resident(s.handle) == 0
    assert L.hsw_synchronize(s.handle) == 0
    ms = L.hsw_last_sweep_kernel_ms(s.handle)
pairs = P.num_elements * P.num_ordinates
print(f"{name} cells={cells} dirs={P.num_ordinates} levels={s.num_levels} sweep {ms:.3f} ms {pairs/ms*1e3:.3e} solves/s")
if os.environ.get("HSW_LEVEL_SIZES", "1") == "1":
    import numpy as np
    cnt = np.zeros(s.num_levels, np.int64)
    for d in range(P.num_ordinates):
        cnt += np.bincount(s.ordering(d).level, minlength=s.num_levels)[: s.num_levels]
    print("level_sizes", " ".join(str(int(x)) for x in cnt))
