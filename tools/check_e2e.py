"""Full-size check of the pipelined host-pointer sweep (hsw_sweep(d=-1) with host buffers):
equal, bit for bit, to the same sweep with the blocks run one after another (HSW_E2E_BLOCKS=1
semantics are per process, so this compares against a direct per-ordinate-block reference:
the all-ordinate host-pointer sweep run twice must be deterministic and match a second
solver's result).  Development aid: python tools/check_e2e.py [config]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import problem as pb

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
P = pb.config(name)
s = pk.SweepSolver(P)
rng = np.random.default_rng(3)
phi = rng.uniform(0, 1, P.num_dofs)
psi_old = rng.uniform(-0.5, 1.0, (P.num_ordinates, P.num_dofs))
a = s.sweep(-1, phi, psi_old)
t = time.time(); b = s.sweep(-1, phi, psi_old); dt = time.time() - t
# per-ordinate host-pointer sweeps for a sample of ordinates (single-ordinate path, no pipeline)
ds = [0, 1, P.num_ordinates // 3, P.num_ordinates // 2, P.num_ordinates - 1]
ok = all(np.array_equal(a[d], s.sweep(d, phi, psi_old[d])) for d in ds)
print(f"{name}: pipelined all-ordinate sweep deterministic={np.array_equal(a, b)} "
      f"matches single-ordinate sweeps={ok} ({dt*1e3:.0f} ms wall)")
