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
FL = os.environ.get("FLAGS")
for flags in ([int(x) for x in FL.split(",")] if FL else [0] if os.environ.get("QUICK") else [0, 1, 2, 4, 3, 5, 6, 7]):
    L.hsw_debug_flags(s.handle, flags)
    for _ in range(2):
        L.hsw_sweep_resident(s.handle); L.hsw_synchronize(s.handle)
    ms = L.hsw_last_sweep_kernel_ms(s.handle)
    print(f"{name} flags={flags} (1 no-faces, 2 no-elim, 4 no-T, 64 no-TMEM-gather, 256 prof-only) sweep {ms:.2f} ms", flush=True)
if os.environ.get("ONLY_FLAGS"): sys.exit(0)

# per-phase clock64 counters (flag 8), cycles per pair as seen by one lane of the pair
import numpy as np
L.hsw_debug_profile.argtypes = [C.c_void_p, C.c_void_p]
L.hsw_debug_flags(s.handle, 8)
L.hsw_sweep_resident(s.handle); L.hsw_synchronize(s.handle)
out = np.zeros(16, np.uint64)
L.hsw_debug_profile(s.handle, C.c_void_p(out.ctypes.data))
n = max(int(out[5]), 1)
names = ["tables", "faces", "assembly", "elimination", "writeback"]
print(name, "pairs", n, " ".join(f"{nm}={int(out[i])/n:.0f}cyc" for i, nm in enumerate(names)), flush=True)
print(name, "panel loop:", " ".join(f"{nm}={int(out[8 + i])/n:.0f}cyc" for i, nm in enumerate([os.environ.get("P8", "wait"), os.environ.get("P9", "U"), "dmma", "factor"])), flush=True)
print(name, "volume split: register tiles", int(out[6]) // n, "cyc, TMEM tiles", int(out[7]) // n, "cyc", flush=True)

for extra in (16, 32):   # only warp 0 / warps 0-3 per CTA work: the single-warp latency of each phase
    L.hsw_debug_flags(s.handle, 8 | extra)
    L.hsw_sweep_resident(s.handle); L.hsw_synchronize(s.handle)
    ms = L.hsw_last_sweep_kernel_ms(s.handle)
    d = np.zeros(16, np.uint64)
    L.hsw_debug_profile(s.handle, C.c_void_p(d.ctypes.data))
    n2 = max(int(d[5]), 1)
    print(name, f"flags 8|{extra}: sweep {ms:.1f} ms, pairs {n2}", " ".join(f"{nm}={int(d[i])/n2:.0f}" for i, nm in enumerate(names)),
          "| factor", int(d[11]) // n2, "gather", int(d[8]) // n2, "update", int(d[9]) // n2, "volT", int(d[7]) // n2,
          "| factor: load", int(d[12]) // n2, "steps", int(d[13]) // n2, "| gather TMEM+reg", int(d[14]) // n2, flush=True)
