"""Generate the golden fixtures of tests/test_golden.py from the CPU oracle.

    python tests/golden/make_golden.py

The oracle (oracle/, the restatement of the reference algorithm pinned to the
reference's own known-answer tests) is run on seeded inputs of small variants
of BASELINE.json's configs; the fixtures freeze its outputs so that (a) the
oracle is regression-pinned bit for bit and (b) the GPU path is checked against
committed vectors without re-running the oracle.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_1810_11080_b200 import problem as pb  # noqa: E402

CASES = {
    "c1": dict(),
    "c2": dict(cells=6, n_mu=2, n_az=8),
    "c3": dict(cells=3, n_mu=2, n_az=4),
    "c4": dict(cells=2, n_mu=2, n_az=4),
    "c5": dict(cells=2, n_mu=2, n_az=4),
}


def inputs(prob, seed):
    rng = np.random.default_rng(seed)
    phi = rng.uniform(0.0, 1.0, prob.num_dofs)
    psi_old = rng.uniform(-0.5, 1.0, (prob.num_ordinates, prob.num_dofs))
    return phi, psi_old


def main():
    O.build()
    for name, kw in CASES.items():
        prob = pb.config(name, **kw)
        orc = O.OracleSolver(prob)
        phi, psi_old = inputs(prob, 2018)
        out = dict(phi=phi, psi_old=psi_old, psi_new=orc.sweep_all(phi, psi_old))
        for d in range(prob.num_ordinates):
            o = orc.ordering(d)
            out[f"order_{d}"] = np.asarray(o["order"], np.int32)
            out[f"lagged_{d}"] = np.asarray(o["lagged_edges"], np.int32)
            out[f"level_{d}"] = np.asarray(o["level"], np.int32)
        if name == "c1":
            si = orc.source_iteration(1e-8, 400, 1)
            out.update(si_phi=si["phi"], si_psi=si["psi"], si_iterations=np.int32(si["iterations"]),
                       si_phi_rel=si["phi_rel"])
        path = os.path.join(HERE, f"{name}_small.npz")
        np.savez_compressed(path, **out)
        print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
