"""Generate tests/golden/ref_*.npz from the REFERENCE ITSELF (test infrastructure).

Runs oracle/_ref/ref_driver — the reference's own headers
(/root/reference/proj/include/hosweep) compiled against the Eigen-subset shim by
`make -C oracle ref` — on seeded 2D problems built by
paper_1810_11080_b200.problem (the same inputs the oracle and the product get),
and stores its outputs: interior faces, per-ordinate couplings / edge weights /
lag flags / orders / cut sets, one lagged sweep of every ordinate, local solves,
direct_oracle, converged source iteration (reference criterion max_d
||dpsi||_inf < tol) and balance_report.

Only runnable where /root/reference exists (this container); the .npz files are
committed and travel to the GPU box.  Usage: python tests/golden/make_ref_golden.py
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1810_11080_b200 import problem as pb  # noqa: E402

DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

# (name, config kwargs, extra problem fields, SI tolerance, SI max iterations, direct_oracle ordinates)
CASES = [
    ("ref_c1", ("c1", {}), {}, 1e-12, 400, 16),
    ("ref_c1_inflow", ("c1", dict(cells=4)), dict(inflow=0.7), 1e-12, 400, 16),
    ("ref_c2_small", ("c2", dict(cells=16, n_mu=2, n_az=8)), {}, 1e-12, 400, 0),
    # the reference's DEFAULT face rule: Romberg (assembly.hpp:33-40, romberg.hpp)
    ("ref_c1_romberg", ("c1", {}), dict(face_rule=1), 1e-12, 400, 16),
    ("ref_c1_romberg_inflow", ("c1", dict(cells=4)), dict(face_rule=1, inflow=0.7), 1e-12, 400, 16),
    ("ref_c2_small_romberg", ("c2", dict(cells=12, n_mu=2, n_az=8)), dict(face_rule=1), 1e-12, 400, 0),
]


def inputs(prob, seed=11):
    rng = np.random.default_rng(seed)
    N = prob.num_dofs
    return (rng.uniform(0.0, 1.0, N), rng.uniform(-0.5, 1.0, (prob.num_ordinates, N)),
            rng.uniform(-1.0, 1.0, prob.block_size))


def run_case(prob, si_tol, si_max, direct_count, face_rule=0):
    phi, psi_old, rhs = inputs(prob)
    ids, st, ss = prob.region_arrays()
    with tempfile.TemporaryDirectory() as tin, tempfile.TemporaryDirectory() as tout:
        arrays = dict(pts=np.asarray(prob.points, np.float64), nodes=np.asarray(prob.element_nodes, np.int32),
                      reg=np.asarray(prob.element_region, np.int32), bf=np.asarray(prob.bfaces, np.int32),
                      w=np.asarray(prob.ord_weight, np.float64), dir=np.asarray(prob.ord_dir, np.float64),
                      ids=ids.astype(np.int32), st=st, ss=ss, src=prob.source_param_array(), phi=phi,
                      psi_old=psi_old, rhs=rhs)
        for k, v in arrays.items():
            np.ascontiguousarray(v).tofile(os.path.join(tin, k))
        meta = [prob.basis_order, prob.geom_order, len(prob.points), prob.num_elements, len(prob.bfaces),
                prob.num_ordinates, len(ids), prob.source_kind, face_rule, prob.face_points, prob.volume_points,
                repr(float(prob.inflow)), repr(si_tol), si_max, direct_count]
        with open(os.path.join(tin, "meta.txt"), "w") as f:
            f.write(" ".join(str(x) for x in meta) + "\n")
        r = subprocess.run([DRIVER, tin, tout], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(r.stderr + r.stdout)
        out = {}
        for line in open(os.path.join(tout, "manifest.txt")):
            name, dt, n = line.split()
            out[name] = np.fromfile(os.path.join(tout, name + ".bin"), dtype=np.dtype(dt))
            assert out[name].size == int(n)
    out.update(phi=phi, psi_old=psi_old, rhs=rhs)
    return out


def main():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    for name, (cfg, kw), extra, tol, mx, ndir in CASES:
        prob = pb.config(cfg, **kw)
        if extra:
            prob = prob.replace(**extra)
        out = run_case(prob, tol, mx, ndir, face_rule=prob.face_rule)
        out["case"] = np.array(repr((cfg, kw, extra, tol, mx, ndir)))
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


if __name__ == "__main__":
    main()
