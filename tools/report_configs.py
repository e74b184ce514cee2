"""Per-config report on one GPU (BASELINE.json configs[0..4]): per-sweep
throughput (device-resident, CUDA events) and source iteration to
||dphi||_2/||phi||_2 < 1e-8 (iterations, device time).  Writes a markdown table.

    python tools/report_configs.py [out.md] [configs...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11080_b200 as pk  # noqa: E402
from paper_1810_11080_b200 import _capi, problem as pb  # noqa: E402


def flops(n):
    return 2.0 / 3.0 * n ** 3 + 2.0 * n * n


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/configs.md"
    names = sys.argv[2:] or ["c1", "c2", "c3", "c4", "c5"]
    L = _capi.load()
    rows = []
    for name in names:
        P = pb.config(name)
        t0 = time.time()
        s = pk.SweepSolver(P, pk.SolveOptions(tolerance=1e-8, max_iterations=2000, criterion="phi_rel_l2"))
        setup = time.time() - t0
        for _ in range(2):
            assert L.hsw_sweep_resident(s.handle) == 0
            assert L.hsw_synchronize(s.handle) == 0
        ms = []
        for _ in range(3):
            L.hsw_sweep_resident(s.handle)
            L.hsw_synchronize(s.handle)
            ms.append(L.hsw_last_sweep_kernel_ms(s.handle))
        m = min(ms)
        pairs = P.num_elements * P.num_ordinates
        state, hist = s.source_iteration(return_psi=False)
        row = dict(config=name, pairs=pairs, n=P.block_size, levels=s.num_levels, setup_s=round(setup, 2),
                   sweep_ms=round(m, 3), solves_per_s=pairs / m * 1e3, tflops=flops(P.block_size) * pairs / m * 1e-9,
                   si_iterations=hist.iterations(), si_converged=hist.converged, si_seconds=round(hist.seconds, 3),
                   si_final_phi_rel=hist.phi_rel[-1] if hist.phi_rel else None)
        rows.append(row)
        print(json.dumps(row), flush=True)
        s.close()
    with open(out, "w") as f:
        f.write("| config | pairs | n | levels | setup s | sweep ms | solves/s | TFLOP/s (LU-alg) | SI iterations to 1e-8 | SI device s |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['config']} | {r['pairs']:,} | {r['n']} | {r['levels']} | {r['setup_s']} | {r['sweep_ms']} | "
                    f"{r['solves_per_s']:.3e} | {r['tflops']:.2f} | {r['si_iterations']}"
                    f"{'' if r['si_converged'] else ' (not converged)'} | {r['si_seconds']} |\n")


if __name__ == "__main__":
    main()
