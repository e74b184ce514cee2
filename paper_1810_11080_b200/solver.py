"""Host-side mirror of the reference's solver interface over the C ABI.

``SweepSolver`` keeps the method names, argument meaning and error behaviour
of ``hosweep::SweepSolver`` (solver.hpp:50-203):

    SweepSolver(problem, options)          ctor: operator + graphs + orderings (solver.hpp:52-78)
    .ordering(d) -> SweepOrdering          solver.hpp:80 (IndexError like std::out_of_range)
    .options                               solver.hpp:81
    .total_lagged_edges()                  solver.hpp:83-87
    .local_solve(e, d, rhs)                solver.hpp:91-93
    .sweep(d, phi, psi_old)                solver.hpp:98-117 (d=-1: all ordinates)
    .direct_oracle(d, phi)                 solver.hpp:121-133
    .source_iteration() -> (SolverState, ConvergenceHistory)   solver.hpp:136-168
    balance_report(solver, state)          solver.hpp:220-245

Vectors are numpy float64 arrays of length N_el*n, element-major (dof m of
element e at e*n + m), one per ordinate — the reference's layout.  Every call
goes through libhosweep_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import _capi
from .problem import Problem

__all__ = [
    "SolveOptions", "SweepOrdering", "SolverState", "ConvergenceHistory", "BalanceReport",
    "SweepSolver", "balance_report", "SolverError", "MeshError", "GeometryError", "AssemblyError",
    "HswError",
]


class HswError(RuntimeError):
    status = -1


class SolverError(HswError):      # solver.hpp:21-23
    status = -5


class MeshError(HswError):        # mesh.hpp:23-25
    status = -2


class GeometryError(HswError):    # mesh.hpp:27-29
    status = -3


class AssemblyError(HswError):    # assembly.hpp:24-26
    status = -4


class LogicError(HswError):       # std::logic_error
    status = -6


class CudaError(HswError):
    status = -8


_STATUS_EXC = {-2: MeshError, -3: GeometryError, -4: AssemblyError, -5: SolverError, -6: LogicError,
               -8: CudaError}


def _raise(rc: int):
    msg = _capi.last_error()
    if rc == -1:
        raise ValueError(msg)
    if rc == -7:
        raise IndexError(msg)
    if rc == -9:
        raise MemoryError(msg)
    raise _STATUS_EXC.get(rc, HswError)(msg)


def _check(rc: int):
    if rc != 0:
        _raise(rc)


def _p(a):
    return a.ctypes.data if a is not None else None


@dataclasses.dataclass
class SolveOptions:
    """solver.hpp:25-32 plus the configs' stopping criterion."""
    tolerance: float = 1e-14
    max_iterations: int = 400
    mode: str = "sweep"            # "sweep" | "direct_oracle"
    weighting: str = "face"        # "unity" | "face" | "siginvface"
    exact_fas_threshold: int = 10
    criterion: str = "psi_linf"    # "psi_linf" (reference) | "phi_rel_l2" (configs)


@dataclasses.dataclass
class SweepOrdering:
    """sweepgraph.hpp:318-325 (+ per-element level of the B200 worklist)."""
    order: np.ndarray
    position: np.ndarray
    lagged_edges: np.ndarray
    lagged_weight: float
    level: np.ndarray

    def is_lagged_position(self, frm: int, to: int) -> bool:
        return bool(self.position[frm] > self.position[to])


@dataclasses.dataclass
class SolverState:
    psi: np.ndarray   # (num_ordinates, N)
    phi: np.ndarray   # (N,)
    iterations: int


@dataclasses.dataclass
class ConvergenceHistory:
    """solver.hpp:34-39 (+ the configs' relative-phi history and the device time)."""
    error: List[float]                 # per iteration, max over ordinates of ||dpsi_d||_inf
    phi_rel: List[float]               # per iteration ||dphi||_2 / ||phi||_2
    converged: bool
    seconds: float = 0.0
    per_ordinate: List[List[float]] = dataclasses.field(default_factory=list)   # error[it][d]

    def iterations(self) -> int:
        return len(self.error)


@dataclasses.dataclass
class BalanceReport:
    source_volume: float
    inflow: float
    source_total: float
    absorption: float
    outflow: float
    net_leakage: float
    residual: float
    outflow_by_attr: Dict[int, float]


_WEIGHT = {"unity": 0, "face": 1, "siginvface": 2, "sig_inv_face": 2}


class SweepSolver:
    def __init__(self, problem: Problem, options: Optional[SolveOptions] = None, device: int = 0,
                 validate_geometry: bool = True, check_local_blocks: bool = True,
                 ordinate_range: Optional[Tuple[int, int]] = None):
        """``ordinate_range=(d0, d1)``: a multi-GPU rank's shard — only those ordinates'
        graphs, orders, worklists and psi are built (sharded.py); all-ordinate calls
        (source_iteration, balance_report, sweep(-1)) then raise IndexError."""
        L = _capi.load()
        self.problem = problem
        self._options = options or SolveOptions()
        self.device = device
        keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a

        pts = arr(problem.points, np.float64)
        nodes = arr(problem.element_nodes, np.int32)
        reg = arr(problem.element_region, np.int32)
        bf = arr(problem.bfaces, np.int32)
        ow = arr(problem.ord_weight, np.float64)
        od = arr(problem.ord_dir, np.float64)
        ids, st, ss = problem.region_arrays()
        ids, st, ss = arr(ids, np.int32), arr(st, np.float64), arr(ss, np.float64)
        d = _capi.hsw_problem_desc()
        d.abi_version = _capi.HSW_ABI_VERSION
        d.dim, d.geom_order, d.basis_order = problem.dim, problem.geom_order, problem.basis_order
        d.num_points, d.points = pts.shape[0], _p(pts)
        d.num_elements, d.element_nodes, d.element_region = nodes.shape[0], _p(nodes), _p(reg)
        d.num_boundary_faces, d.boundary_faces = bf.shape[0], _p(bf)
        d.num_ordinates, d.ordinate_weight, d.ordinate_dir = ow.shape[0], _p(ow), _p(od)
        d.num_regions, d.region_ids, d.sigma_t, d.sigma_s = len(ids), _p(ids), _p(st), _p(ss)
        d.source_kind = problem.source_kind
        for i, v in enumerate(problem.source_param_array()):
            d.source_params[i] = v
        d.inflow = problem.inflow
        d.volume_points, d.face_points = problem.volume_points, problem.face_points
        d.weighting = _WEIGHT[self._options.weighting]
        d.exact_fas_threshold = self._options.exact_fas_threshold
        d.validate_geometry = int(validate_geometry)
        # the reference constructor factors every local block and throws SolverError
        # for a singular one (solver.hpp:67-75): on by default here too
        d.check_local_blocks = int(check_local_blocks)
        d.device = device  # < 0: host-only plan (graphs/orderings, no device state)
        d.face_rule = int(getattr(problem, "face_rule", 0))
        d.romberg_tol = float(getattr(problem, "romberg_tol", 1e-10))
        d.romberg_max_levels = int(getattr(problem, "romberg_max_levels", 16))
        d.romberg_min_levels = int(getattr(problem, "romberg_min_levels", 6))
        if ordinate_range is not None:
            d.ordinate_begin, d.ordinate_end = int(ordinate_range[0]), int(ordinate_range[1])
        self.ordinate_range = tuple(ordinate_range) if ordinate_range is not None else (0, problem.num_ordinates)
        h = C.c_void_p()
        _check(L.hsw_create(C.byref(d), C.byref(h)))
        self._h = h
        sz = np.zeros(6, np.int64)
        _check(L.hsw_sizes(self._h, _p(sz)))
        self.num_elements, self.block_size, self.num_ordinates, self.num_dofs = (int(x) for x in sz[:4])
        self.num_interior_faces, self.num_levels = int(sz[4]), int(sz[5])

    def close(self):
        if getattr(self, "_h", None):
            _capi.load().hsw_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def options(self) -> SolveOptions:
        return self._options

    # ---- graph / ordering introspection (sweepgraph.hpp:318-325)
    def ordering(self, d: int) -> SweepOrdering:
        L = _capi.load()
        n = self.num_elements
        order = np.zeros(n, np.int32)
        pos = np.zeros(n, np.int32)
        lev = np.zeros(n, np.int32)
        nl = C.c_int()
        w = C.c_double()
        _check(L.hsw_ordering(self._h, d, _p(order), _p(pos), None, 0, C.byref(nl), C.byref(w), _p(lev)))
        lag = np.zeros(max(nl.value, 1), np.int32)
        _check(L.hsw_ordering(self._h, d, None, None, _p(lag), nl.value, None, None, None))
        return SweepOrdering(order, pos, lag[: nl.value], w.value, lev)

    @property
    def pivot_fallbacks(self) -> int:
        """Calls redone with the partial-pivoting kernel because the static-pivot tile LU refused a
        local block (0 on the BASELINE.json configs; the handle keeps to the pivoted kernel after)."""
        return int(_capi.load().hsw_pivot_fallbacks(self._h))

    def total_lagged_edges(self) -> int:
        out = C.c_int64()
        _check(_capi.load().hsw_total_lagged_edges(self._h, C.byref(out)))
        return out.value

    def couplings(self, d: int) -> Tuple[np.ndarray, np.ndarray]:
        """(face, downwind, upwind, lagged) per coupling and the edge weights."""
        L = _capi.load()
        cnt = C.c_int()
        _check(L.hsw_couplings(self._h, d, None, None, 0, C.byref(cnt)))
        ints = np.zeros((max(cnt.value, 1), 4), np.int32)
        w = np.zeros(max(cnt.value, 1))
        _check(L.hsw_couplings(self._h, d, _p(ints), _p(w), cnt.value, None))
        return ints[: cnt.value], w[: cnt.value]

    def interior_faces(self) -> np.ndarray:
        L = _capi.load()
        cnt = C.c_int()
        _check(L.hsw_interior_faces(self._h, None, 0, C.byref(cnt)))
        out = np.zeros((max(cnt.value, 1), 5), np.int32)
        _check(L.hsw_interior_faces(self._h, _p(out), cnt.value, None))
        return out[: cnt.value]

    # ---- solves
    def local_solve(self, e: int, d: int, rhs) -> np.ndarray:
        rhs = np.ascontiguousarray(rhs, np.float64)
        out = np.zeros(self.block_size)
        _check(_capi.load().hsw_local_solve(self._h, e, d, _p(rhs), _p(out)))
        return out

    def sweep(self, d: int, phi, psi_old, out: Optional[np.ndarray] = None) -> np.ndarray:
        """solver.hpp:98-117.  d = -1 sweeps every ordinate (psi_old / the result are
        (num_ordinates, num_dofs)).  ``out`` (optional, C-contiguous float64 of psi_old's
        shape, not aliasing it) receives the result instead of a freshly allocated array:
        a fresh multi-GB array pays the OS's first-touch page faults on every call."""
        self._last_si_state = None   # the device psi buffers are reused by this call
        phi = np.ascontiguousarray(phi, np.float64)
        psi_old = np.ascontiguousarray(psi_old, np.float64)
        if out is None:
            out = np.zeros_like(psi_old)
        elif (out.dtype != np.float64 or out.shape != psi_old.shape or not out.flags.c_contiguous
              or np.shares_memory(out, psi_old)):
            raise ValueError("sweep: out must be a C-contiguous float64 array of psi_old's shape, not aliasing it")
        _check(_capi.load().hsw_sweep(self._h, d, _p(phi), _p(psi_old), _p(out)))
        return out

    def direct_oracle(self, d: int, phi) -> np.ndarray:
        self._last_si_state = None
        phi = np.ascontiguousarray(phi, np.float64)
        out = np.zeros(self.num_dofs)
        _check(_capi.load().hsw_direct_oracle(self._h, d, _p(phi), _p(out)))
        return out

    def source_iteration(self, return_psi: bool = True):
        o = self._options
        opts = _capi.hsw_si_options(o.tolerance, o.max_iterations,
                                    0 if o.criterion == "psi_linf" else 1,
                                    0 if o.mode == "sweep" else 1)
        res = _capi.hsw_si_result()
        psi = np.zeros((self.num_ordinates, self.num_dofs)) if return_psi else None
        phi = np.zeros(self.num_dofs)
        eh = np.zeros(max(o.max_iterations, 1))
        ph = np.zeros(max(o.max_iterations, 1))
        po = np.zeros((max(o.max_iterations, 1), self.num_ordinates))
        _check(_capi.load().hsw_source_iteration(self._h, C.byref(opts), C.byref(res), _p(psi), _p(phi),
                                                 _p(eh), _p(ph), _p(po)))
        it = res.iterations
        state = SolverState(psi, phi, it)
        self._last_si_state = state   # resident on the device until the next call that moves psi
        hist = ConvergenceHistory(list(eh[:it]), list(ph[:it]), bool(res.converged), res.seconds,
                                  [list(r) for r in po[:it]])
        return state, hist

    @staticmethod
    def zero_block_at_create_for_test(e: int, d: int):
        """test_solver.cpp:332-344 for the constructor: the next SweepSolver created on
        this thread has the (e, d) local block zeroed from the start."""
        _check(_capi.load().hsw_debug_create_zero_block(e, d))

    def zero_block_for_test(self, e: int, d: int):
        """test_solver.cpp:332-344 hook: the (e, d) local block is zeroed."""
        _check(_capi.load().hsw_debug_zero_block(self._h, e, d))


def balance_report(solver: SweepSolver, state: Optional[SolverState] = None) -> BalanceReport:
    """solver.hpp:220-245 conservation functionals of a state."""
    out = np.zeros(5)
    attrs = np.zeros(64, np.int32)
    vals = np.zeros(64)
    cnt = C.c_int()
    if state is None or state is getattr(solver, "_last_si_state", None) or state.psi is None:
        # the solver's own converged state is still resident on the device: evaluate there
        # (hsw_balance_resident), no 2 x nd x N host round trip
        _check(_capi.load().hsw_balance_resident(solver.handle, _p(out), _p(attrs), _p(vals), 64, C.byref(cnt)))
    else:
        psi = np.ascontiguousarray(state.psi, np.float64)
        phi = np.ascontiguousarray(state.phi, np.float64)
        _check(_capi.load().hsw_balance(solver.handle, _p(psi), _p(phi), _p(out), _p(attrs), _p(vals), 64,
                                        C.byref(cnt)))
    by = {int(attrs[i]): float(vals[i]) for i in range(min(cnt.value, 64))}
    return BalanceReport(out[0], out[1], out[0] + out[1], out[2], out[3], out[3] - out[1], out[4], by)
