"""Test-only shard backend over the CPU oracle (NOT product code).

It gives the collective driver (paper_1810_11080_b200/sharded.py) a CPU data
path so the world_size-2 gloo tests exercise the exact control flow the GPU
ranks run.  Arithmetic mirrors orc::Oracle::source_iteration
(oracle/hosweep_oracle.cpp): phi accumulated as ph += w * psi in increasing d
(no FMA), sequential norm sums, so a one-rank run reproduces the oracle's own
source iteration bit for bit.
"""
import numpy as np
import torch

import oracle as O


class OracleShardBackend:
    def __init__(self, problem):
        self.o = O.OracleSolver(problem)
        self.w = np.asarray(problem.ord_weight, np.float64)
        self.num_ordinates = problem.num_ordinates
        self.num_dofs = problem.num_dofs
        self.device = torch.device("cpu")
        self.reset()

    def zeros(self):
        return torch.zeros(self.num_dofs, dtype=torch.float64)

    def reset(self):
        self.psi_old = np.zeros((self.num_ordinates, self.num_dofs))
        self.psi_new = np.zeros((self.num_ordinates, self.num_dofs))

    def sweep(self, d0, d1, phi):
        ph = phi.numpy()
        for d in range(d0, d1):
            self.psi_new[d] = self.o.sweep(d, ph, self.psi_old[d])

    def phi_partial(self, d0, d1, prefix, out):
        ph = prefix.numpy().copy() if prefix is not None else np.zeros(self.num_dofs)
        for d in range(d0, d1):
            ph = ph + self.w[d] * self.psi_new[d]
        out.copy_(torch.from_numpy(ph))

    def psi_error(self, d0, d1):
        return float(np.abs(self.psi_new[d0:d1] - self.psi_old[d0:d1]).max())

    def phi_norms(self, phi_new, phi_old):
        a, b = phi_new.numpy(), phi_old.numpy()
        df = a - b
        return float(np.cumsum(df * df)[-1]), float(np.cumsum(a * a)[-1])

    def advance(self, phi):
        self.psi_old, self.psi_new = self.psi_new, self.psi_old

    def psi(self, d0, d1):
        return self.psi_old[d0:d1].copy()
