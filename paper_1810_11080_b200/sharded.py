"""Direction-sharded source iteration over ranks.

``SweepSolver::source_iteration`` (solver.hpp:136-168) sweeps every ordinate
independently with a shared scalar flux phi, then forms phi = sum_d w_d psi_d
(in increasing d, from zero) and the error max_d ||psi_new_d - psi_old_d||_inf.
So the ordinates shard with no data-path exchange inside a sweep; one process
per GPU (torch.distributed: NCCL over NVLink on the B200 box, gloo in the CPU
tests) owns a contiguous ordinate block [d0, d1) and keeps only its psi.

Per iteration:
  1. every rank sweeps its block with the same phi (device-resident psi, the
     B200 sweep kernels through ``hsw_shard_sweep``);
  2. phi is a *chained prefix in ordinate order*: rank r receives the partial
     sum of the ordinates < d0_r from rank r-1, adds its block in ascending d
     with the single-device FMA chain (``hsw_shard_phi_partial``) and sends the
     result on; the last rank broadcasts phi.  phi is therefore bit-identical to
     the single-device ``hsw_source_iteration`` (and to any other rank count);
  3. the psi error is an all-reduce MAX of the block maxima (exact);
  4. the phi-relative change uses the same reduction tree on the identical phi
     on every rank (``hsw_shard_phi_norms``), so every rank takes the same
     convergence decision.
The exchange is an (N-1)-hop chain plus one broadcast of N_el*n doubles
(C4: 16.8 MB) and one scalar all-reduce per iteration.

The driver talks to a *backend* (``DeviceShardBackend`` for the library; the
CPU tests inject an oracle-backed one) so the collective logic is one code path.
A rank creates its solver with ``SweepSolver(prob, device=local,
ordinate_range=block_of(nd, rank, world))``: only its block's graphs, orders,
worklists and psi are built (the element tensors are shared by all ordinates).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import time
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from .solver import SweepSolver, _check


def block_of(num_ordinates: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous ordinate block of ``rank`` (sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"rank {rank} of world {world}")
    if world > num_ordinates:
        raise ValueError(f"{world} ranks for {num_ordinates} ordinates: every rank needs an ordinate")
    return (rank * num_ordinates) // world, ((rank + 1) * num_ordinates) // world


class DeviceShardBackend:
    """Per-rank device primitives of ``include/hosweep_b200.h`` (hsw_shard_*)."""

    def __init__(self, solver: SweepSolver):
        if getattr(solver, "device", 0) < 0:
            raise RuntimeError("DeviceShardBackend needs a device solver (device >= 0); no CPU fallback")
        self.solver = solver
        self.L = _capi.load()
        self.h = solver.handle
        self.num_ordinates = solver.num_ordinates
        self.num_dofs = solver.num_dofs
        self.device = torch.device("cuda", solver.device)
        self._stream = torch.cuda.ExternalStream(self.L.hsw_stream(self.h), device=self.device)

    # torch work (collectives, allocations) and the library stream are ordered by
    # explicit synchronisation at the hand-over points
    def _lib_after_torch(self):
        torch.cuda.current_stream(self.device).synchronize()

    def _torch_after_lib(self):
        self._stream.synchronize()

    def zeros(self) -> torch.Tensor:
        return torch.zeros(self.num_dofs, dtype=torch.float64, device=self.device)

    def reset(self):
        _check(self.L.hsw_shard_reset(self.h))

    def sweep(self, d0: int, d1: int, phi: torch.Tensor):
        self._lib_after_torch()
        _check(self.L.hsw_shard_sweep(self.h, d0, d1, phi.data_ptr()))

    def phi_partial(self, d0: int, d1: int, prefix: Optional[torch.Tensor], out: torch.Tensor):
        self._lib_after_torch()
        _check(self.L.hsw_shard_phi_partial(self.h, d0, d1, prefix.data_ptr() if prefix is not None else None,
                                            out.data_ptr()))
        self._torch_after_lib()

    def psi_error(self, d0: int, d1: int) -> float:
        v = C.c_double()
        _check(self.L.hsw_shard_psi_error(self.h, d0, d1, C.byref(v)))
        return v.value

    def phi_norms(self, phi_new: torch.Tensor, phi_old: torch.Tensor) -> Tuple[float, float]:
        self._lib_after_torch()
        out = np.zeros(2)
        _check(self.L.hsw_shard_phi_norms(self.h, phi_new.data_ptr(), phi_old.data_ptr(), out.ctypes.data))
        return float(out[0]), float(out[1])

    def advance(self, phi: torch.Tensor):
        self._lib_after_torch()
        _check(self.L.hsw_shard_advance(self.h, phi.data_ptr()))
        self._torch_after_lib()

    def psi(self, d0: int, d1: int) -> np.ndarray:
        out = np.empty((d1 - d0, self.num_dofs))
        _check(self.L.hsw_shard_psi(self.h, d0, d1, out.ctypes.data))
        return out


@dataclasses.dataclass
class ShardedResult:
    iterations: int
    converged: bool
    final_error: float
    final_phi_rel: float
    errors: List[float]
    phi_rels: List[float]
    seconds: float
    phi: np.ndarray                 # identical on every rank
    blocks: List[Tuple[int, int]]   # the ordinate blocks this rank swept
    psi: Optional[np.ndarray]       # this rank's blocks' psi (ordinate-major), if requested


def _world(group) -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def sharded_source_iteration(backend, tolerance: float = 1e-14, max_iterations: int = 400,
                             criterion: str = "psi_linf", group=None, local_blocks: Optional[int] = None,
                             return_psi: bool = False) -> ShardedResult:
    """Source iteration with the ordinates sharded over the ranks of ``group``.

    The stopping defaults are the reference's SolveOptions (solver.hpp:25-32:
    tolerance 1e-14 on max_d ||dpsi_d||_inf, 400 iterations), the same as
    ``SweepSolver.source_iteration``; pass ``tolerance=1e-8,
    criterion="phi_rel_l2"`` for the configs' relative-phi criterion.

    ``local_blocks`` (single rank only) splits the ordinates into that many
    blocks handled in sequence by this process with the same chained phi: the
    single-GPU check that block sweeps + chained partial sums reproduce the
    unsharded iteration bit for bit.
    """
    if criterion not in ("phi_rel_l2", "psi_linf"):
        raise ValueError(f"criterion {criterion!r}")
    rank, world = _world(group)
    nd = backend.num_ordinates
    if local_blocks is not None:
        if world != 1:
            raise ValueError("local_blocks is a single-rank check")
        blocks = [block_of(nd, b, local_blocks) for b in range(local_blocks)]
    else:
        blocks = [block_of(nd, rank, world)]
    peer = lambda r: dist.get_global_rank(group, r) if group is not None else r  # noqa: E731

    backend.reset()
    phi = backend.zeros()
    errors: List[float] = []
    rels: List[float] = []
    converged = False
    err = rel = float("nan")
    t0 = time.perf_counter()
    it = 0
    for it in range(1, max_iterations + 1):
        for a, b in blocks:
            backend.sweep(a, b, phi)
        err = max(backend.psi_error(a, b) for a, b in blocks)
        # phi: chained prefix sum in ordinate order (bit-identical to one device)
        prefix = None
        if world > 1 and rank > 0:
            prefix = backend.zeros()
            dist.recv(prefix, src=peer(rank - 1), group=group)
        for a, b in blocks:
            out = backend.zeros()
            backend.phi_partial(a, b, prefix, out)
            prefix = out
        phi_new = prefix
        if world > 1:
            if rank < world - 1:
                dist.send(phi_new, dst=peer(rank + 1), group=group)
            dist.broadcast(phi_new, src=peer(world - 1), group=group)
            e = torch.tensor([err], dtype=torch.float64, device=phi_new.device)
            dist.all_reduce(e, op=dist.ReduceOp.MAX, group=group)
            err = float(e.item())
        num, den = backend.phi_norms(phi_new, phi)
        rel = math.sqrt(num) / math.sqrt(den) if den > 0.0 else (math.inf if num > 0.0 else 0.0)
        backend.advance(phi_new)
        phi = phi_new
        errors.append(err)
        rels.append(rel)
        if (err if criterion == "psi_linf" else rel) < tolerance:
            converged = True
            break
    seconds = time.perf_counter() - t0
    psi = np.concatenate([backend.psi(a, b) for a, b in blocks]) if return_psi else None
    return ShardedResult(it, converged, err, rel, errors, rels, seconds,
                         phi.detach().cpu().numpy().copy(), blocks, psi)
