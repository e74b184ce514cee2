"""Ablation timing of the sweep kernel phases (development aid, results are NOT valid solves)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import problem as pb, _capi
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
P = pb.config(name)
s = pk.SweepSolver(P)
L = _capi.load()
L.hsw_debug_flags.argtypes = [C.c_void_p, C.c_int]
for flags in [0, 1, 2, 4, 3, 5, 6, 7]:
    L.hsw_debug_flags(s.handle, flags)
    for _ in range(2):
        L.hsw_sweep_resident(s.handle); L.hsw_synchronize(s.handle)
    ms = L.hsw_last_sweep_kernel_ms(s.handle)
    print(f"{name} flags={flags} (1 no-faces, 2 no-elim, 4 no-T) sweep {ms:.2f} ms", flush=True)
