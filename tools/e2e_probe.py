"""e2e through SweepSolver.sweep (pageable numpy) vs pinned hsw_sweep (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import problem as pb
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
P = pb.config(name)
s = pk.SweepSolver(P)
N, nd = P.num_dofs, P.num_ordinates
phi = np.full(N, 0.1)
psi = np.zeros((nd, N))
psi = s.sweep(-1, phi, psi)
for k in range(3):
    t = time.perf_counter()
    psi = s.sweep(-1, phi, psi)
    print(f"{name} pageable fresh-output sweep {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
out = np.empty_like(psi)
out[:] = 0
from paper_1810_11080_b200 import _capi
import ctypes as C
L = _capi.load()
for k in range(2):
    t = time.perf_counter()
    assert L.hsw_sweep(s.handle, -1, phi.ctypes.data, psi.ctypes.data, out.ctypes.data) == 0
    print(f"{name} pageable reused-output sweep {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
