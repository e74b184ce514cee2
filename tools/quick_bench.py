"""Quick per-config sweep timing (development aid; bench.py is the contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import problem as pb, _capi

def flops(n): return 2.0 / 3.0 * n ** 3 + 2.0 * n * n

for name in (sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]):
    t = time.time()
    P = pb.config(name)
    s = pk.SweepSolver(P)
    setup = time.time() - t
    L = _capi.load()
    for _ in range(2):
        assert L.hsw_sweep_resident(s.handle) == 0
        assert L.hsw_synchronize(s.handle) == 0
    ms = []
    for _ in range(3):
        L.hsw_sweep_resident(s.handle); L.hsw_synchronize(s.handle)
        ms.append(L.hsw_last_sweep_kernel_ms(s.handle))
    m = min(ms)
    pairs = P.num_elements * P.num_ordinates
    n = P.block_size
    print(f"{name}: setup {setup:.1f}s levels {s.num_levels} sweep {m:.3f} ms  {pairs/m*1e3:.3e} solves/s  "
          f"{flops(n)*pairs/m*1e-9:.2f} TFLOP/s(LU-alg)  launches {L.hsw_last_launch_count(s.handle)} pivot_fallbacks {L.hsw_pivot_fallbacks(s.handle)}", flush=True)
    s.close()
