import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import problem as pb, _capi
for name, kw in [("c1", dict(cells=2)), ("c2", dict(cells=2, n_mu=2, n_az=4)), ("c3", dict(cells=2, n_mu=2, n_az=4)),
                 ("c4", dict(cells=2, n_mu=2, n_az=4)), ("c5", dict(cells=2, n_mu=2, n_az=4))]:
    P = pb.config(name, **kw)
    try:
        s = pk.SweepSolver(P)
        o = O.OracleSolver(P)
        rng = np.random.default_rng(1)
        errs = []
        for e in range(min(2, P.num_elements)):
            for d in range(2):
                rhs = rng.uniform(-1, 1, P.block_size)
                x = s.local_solve(e, d, rhs)
                A = o.diag_block(e, d)
                errs.append(np.abs(A @ x - rhs).max())
        print(name, "n", P.block_size, "local residual", max(errs), flush=True)
    except Exception as ex:
        print(name, "ERROR", type(ex).__name__, str(ex)[:300], flush=True)
