"""ctypes binding of the CPU oracle (oracle/hosweep_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py, never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "libhosweep_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "hosweep_oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE], env=dict(os.environ, CXX="g++"))
    return _LIB_PATH


class orc_problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("geom_order", C.c_int), ("basis_order", C.c_int),
        ("num_points", C.c_int), ("points", C.c_void_p),
        ("num_elements", C.c_int), ("element_nodes", C.c_void_p), ("element_region", C.c_void_p),
        ("num_bfaces", C.c_int), ("bfaces", C.c_void_p),
        ("num_ordinates", C.c_int), ("ord_weight", C.c_void_p), ("ord_dir", C.c_void_p),
        ("num_regions", C.c_int), ("region_ids", C.c_void_p), ("sigma_t", C.c_void_p),
        ("sigma_s", C.c_void_p),
        ("source_kind", C.c_int), ("source_params", C.c_double * 8), ("inflow", C.c_double),
        ("volume_points", C.c_int), ("face_points", C.c_int),
        ("weighting", C.c_int), ("fas_threshold", C.c_int),
        ("validate_geometry", C.c_int), ("cache_lu", C.c_int), ("check_rcond", C.c_int),
        ("num_active", C.c_int), ("active", C.c_void_p),
        ("face_rule", C.c_int), ("romberg_tol", C.c_double), ("romberg_max_levels", C.c_int),
        ("romberg_min_levels", C.c_int),
    ]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        vp, ip, dp, cp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_char_p
        L.orc_create.restype = vp
        L.orc_create.argtypes = [C.POINTER(orc_problem), cp, C.c_int]
        L.orc_create_with_zero_block.restype = vp
        L.orc_create_with_zero_block.argtypes = [C.POINTER(orc_problem), C.c_int, C.c_int, cp, C.c_int]
        L.orc_destroy.argtypes = [vp]
        for f in ("orc_block_size", "orc_face_nodes", "orc_num_interior_faces"):
            getattr(L, f).argtypes = [vp]
            getattr(L, f).restype = C.c_int
        L.orc_interior_faces.argtypes = [vp, vp]
        L.orc_num_couplings.argtypes = [vp, C.c_int]
        L.orc_num_lagged.argtypes = [vp, C.c_int]
        L.orc_couplings.argtypes = [vp, C.c_int, vp, vp]
        L.orc_coupling_block.argtypes = [vp, C.c_int, C.c_int, vp]
        L.orc_ordering.argtypes = [vp, C.c_int, vp, vp, vp, vp]
        L.orc_ordering.restype = C.c_double
        L.orc_mass.argtypes = [vp, C.c_int, vp, vp]
        L.orc_source.argtypes = [vp, C.c_int, vp, vp]
        L.orc_diag_block.argtypes = [vp, C.c_int, C.c_int, vp]
        L.orc_local_solve.argtypes = [vp, C.c_int, C.c_int, vp, vp, cp, C.c_int]
        L.orc_sweep.argtypes = [vp, C.c_int, vp, vp, vp, cp, C.c_int]
        L.orc_sweep_all.argtypes = [vp, vp, vp, vp, cp, C.c_int]
        L.orc_sweep_subset.argtypes = [vp, C.c_int, vp, vp, vp, cp, C.c_int]
        L.orc_direct_oracle.argtypes = [vp, C.c_int, vp, vp, cp, C.c_int]
        L.orc_sweep_sample.argtypes = [vp, C.c_int, vp, C.c_int, vp, cp, C.c_int]
        L.orc_sweep_sample.restype = C.c_longlong
        L.orc_source_iteration.argtypes = [vp, C.c_double, C.c_int, C.c_int, vp, vp, vp, vp, vp, cp, C.c_int]
        L.orc_balance.argtypes = [vp, vp, vp, vp, vp, vp, C.c_int]
        L.orc_graph_tarjan.argtypes = [C.c_int, C.c_int, vp, vp]
        L.orc_graph_order.argtypes = [C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp]
        L.orc_graph_order.restype = C.c_double
        L.orc_gauss_legendre.argtypes = [C.c_int, vp, vp]
        L.orc_gauss_lobatto.argtypes = [C.c_int, vp]
        L.orc_basis_eval.argtypes = [C.c_int, C.c_int, vp, vp, vp]
        L.orc_face_geometry.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_double, vp]
        L.orc_jacobian.argtypes = [vp, C.c_int, vp, vp]
        L.orc_jacobian.restype = C.c_double
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data if a is not None else None


class OracleError(RuntimeError):
    pass


class OracleSolver:
    """CPU restatement of ``hosweep::SweepSolver`` (solver.hpp:50-203) over an
    assembled operator (assembly.hpp:333-409)."""

    def __init__(self, prob, cache_lu: bool = True, validate: bool = True, check_rcond: bool = True,
                 zero_block: Optional[tuple] = None, active=None):
        L = lib()
        self.prob = prob
        keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a

        pts = arr(prob.points, np.float64)
        nodes = arr(prob.element_nodes, np.int32)
        reg = arr(prob.element_region, np.int32)
        bf = arr(prob.bfaces, np.int32)
        ow = arr(prob.ord_weight, np.float64)
        od = arr(prob.ord_dir, np.float64)
        ids, st, ss = prob.region_arrays()
        ids, st, ss = arr(ids, np.int32), arr(st, np.float64), arr(ss, np.float64)
        s = orc_problem()
        s.dim, s.geom_order, s.basis_order = prob.dim, prob.geom_order, prob.basis_order
        s.num_points, s.points = pts.shape[0], _p(pts)
        s.num_elements, s.element_nodes, s.element_region = nodes.shape[0], _p(nodes), _p(reg)
        s.num_bfaces, s.bfaces = bf.shape[0], _p(bf)
        s.num_ordinates, s.ord_weight, s.ord_dir = ow.shape[0], _p(ow), _p(od)
        s.num_regions, s.region_ids, s.sigma_t, s.sigma_s = len(ids), _p(ids), _p(st), _p(ss)
        s.source_kind = prob.source_kind
        for i, v in enumerate(prob.source_param_array()):
            s.source_params[i] = v
        s.inflow = prob.inflow
        s.volume_points, s.face_points = prob.volume_points, prob.face_points
        s.weighting, s.fas_threshold = prob.weighting, prob.fas_threshold
        s.face_rule = int(getattr(prob, "face_rule", 0))
        s.romberg_tol = float(getattr(prob, "romberg_tol", 1e-10))
        s.romberg_max_levels = int(getattr(prob, "romberg_max_levels", 16))
        s.romberg_min_levels = int(getattr(prob, "romberg_min_levels", 6))
        s.validate_geometry, s.cache_lu, s.check_rcond = int(validate), int(cache_lu), int(check_rcond)
        if active is not None:
            act = arr(active, np.int32)
            s.num_active, s.active = len(act), _p(act)
        err = C.create_string_buffer(1024)
        if zero_block is not None:
            h = L.orc_create_with_zero_block(C.byref(s), zero_block[0], zero_block[1], err, 1024)
        else:
            h = L.orc_create(C.byref(s), err, 1024)
        if not h:
            raise OracleError(err.value.decode())
        self.h = h
        self.nb = L.orc_block_size(h)
        self.nfn = L.orc_face_nodes(h)
        self.nel = prob.num_elements
        self.nd = prob.num_ordinates
        self.N = self.nel * self.nb

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def _check(self, rc, err):
        if rc != 0:
            raise OracleError(err.value.decode())

    def interior_faces(self) -> np.ndarray:
        n = lib().orc_num_interior_faces(self.h)
        out = np.zeros((n, 5), np.int32)
        lib().orc_interior_faces(self.h, _p(out))
        return out

    def couplings(self, d: int):
        """(face, downwind, upwind, lagged) int array and face weights."""
        n = lib().orc_num_couplings(self.h, d)
        ints = np.zeros((n, 4), np.int32)
        w = np.zeros(n)
        lib().orc_couplings(self.h, d, _p(ints), _p(w))
        return ints, w

    def coupling_block(self, d: int, c: int) -> np.ndarray:
        out = np.zeros((self.nfn, self.nfn))
        lib().orc_coupling_block(self.h, d, c, _p(out))
        return out

    def ordering(self, d: int):
        """dict(order, position, lagged_edges, lagged_weight, level)."""
        nl = lib().orc_num_lagged(self.h, d)
        order = np.zeros(self.nel, np.int32)
        pos = np.zeros(self.nel, np.int32)
        lag = np.zeros(max(nl, 1), np.int32)
        lev = np.zeros(self.nel, np.int32)
        w = lib().orc_ordering(self.h, d, _p(order), _p(pos), _p(lag), _p(lev))
        return dict(order=order, position=pos, lagged_edges=lag[:nl], lagged_weight=w, level=lev)

    def total_lagged_edges(self) -> int:
        return sum(lib().orc_num_lagged(self.h, d) for d in range(self.nd))

    def mass(self, e: int):
        mt = np.zeros((self.nb, self.nb))
        ms = np.zeros((self.nb, self.nb))
        lib().orc_mass(self.h, e, _p(mt), _p(ms))
        return mt, ms

    def source(self, d: int):
        v = np.zeros(self.N)
        b = np.zeros(self.N)
        lib().orc_source(self.h, d, _p(v), _p(b))
        return v, b

    def diag_block(self, e: int, d: int) -> np.ndarray:
        A = np.zeros((self.nb, self.nb))
        lib().orc_diag_block(self.h, e, d, _p(A))
        return A

    def local_solve(self, e: int, d: int, rhs) -> np.ndarray:
        rhs = np.ascontiguousarray(rhs, np.float64)
        out = np.zeros(self.nb)
        err = C.create_string_buffer(1024)
        self._check(lib().orc_local_solve(self.h, e, d, _p(rhs), _p(out), err, 1024), err)
        return out

    def sweep(self, d: int, phi, psi_old) -> np.ndarray:
        phi = np.ascontiguousarray(phi, np.float64)
        psi_old = np.ascontiguousarray(psi_old, np.float64)
        out = np.zeros(self.N)
        err = C.create_string_buffer(1024)
        self._check(lib().orc_sweep(self.h, d, _p(phi), _p(psi_old), _p(out), err, 1024), err)
        return out

    def sweep_all(self, phi, psi_old) -> np.ndarray:
        phi = np.ascontiguousarray(phi, np.float64)
        psi_old = np.ascontiguousarray(psi_old, np.float64).reshape(self.nd, self.N)
        out = np.zeros((self.nd, self.N))
        err = C.create_string_buffer(1024)
        self._check(lib().orc_sweep_all(self.h, _p(phi), _p(psi_old), _p(out), err, 1024), err)
        return out

    def sweep_subset(self, ds, phi) -> np.ndarray:
        ds = np.ascontiguousarray(ds, np.int32)
        phi = np.ascontiguousarray(phi, np.float64)
        out = np.zeros((len(ds), self.N))
        err = C.create_string_buffer(1024)
        self._check(lib().orc_sweep_subset(self.h, len(ds), _p(ds), _p(phi), _p(out), err, 1024), err)
        return out

    def sweep_sample(self, ds, max_elems: int, phi) -> int:
        """Bounded CPU-baseline sample: the first max_elems elements of each
        listed ordinate's sweep (on-the-fly local assembly + LU); returns solves."""
        ds = np.ascontiguousarray(ds, np.int32)
        phi = np.ascontiguousarray(phi, np.float64)
        err = C.create_string_buffer(1024)
        n = lib().orc_sweep_sample(self.h, len(ds), _p(ds), max_elems, _p(phi), err, 1024)
        if n < 0:
            raise OracleError(err.value.decode())
        return int(n)

    def direct_oracle(self, d: int, phi) -> np.ndarray:
        phi = np.ascontiguousarray(phi, np.float64)
        out = np.zeros(self.N)
        err = C.create_string_buffer(1024)
        self._check(lib().orc_direct_oracle(self.h, d, _p(phi), _p(out), err, 1024), err)
        return out

    def source_iteration(self, tol: float = 1e-14, max_iterations: int = 400, criterion: int = 0):
        """Returns dict(psi (nd,N), phi (N), error (it,), phi_rel (it,), converged)."""
        psi = np.zeros((self.nd, self.N))
        phi = np.zeros(self.N)
        eh = np.zeros(max_iterations)
        ph = np.zeros(max_iterations)
        conv = np.zeros(1, np.int32)
        err = C.create_string_buffer(1024)
        it = lib().orc_source_iteration(self.h, tol, max_iterations, criterion, _p(psi), _p(phi),
                                        _p(eh), _p(ph), _p(conv), err, 1024)
        if it < 0:
            raise OracleError(err.value.decode())
        return dict(psi=psi, phi=phi, error=eh[:it], phi_rel=ph[:it], converged=bool(conv[0]),
                    iterations=it)

    def balance(self, psi, phi):
        psi = np.ascontiguousarray(psi, np.float64)
        phi = np.ascontiguousarray(phi, np.float64)
        out = np.zeros(5)
        attrs = np.zeros(16, np.int32)
        vals = np.zeros(16)
        k = lib().orc_balance(self.h, _p(psi), _p(phi), _p(out), _p(attrs), _p(vals), 16)
        return dict(source_volume=out[0], inflow=out[1], absorption=out[2], outflow=out[3],
                    residual=out[4], source_total=out[0] + out[1],
                    outflow_by_attr={int(attrs[i]): float(vals[i]) for i in range(k)})

    def face_geometry(self, e, f, s, t=0.0):
        out = np.zeros(7)
        lib().orc_face_geometry(self.h, e, f, s, t, _p(out))
        return out[:3], out[3:6], out[6]

    def jacobian(self, e, xi):
        xi3 = np.zeros(3)
        xi3[: len(xi)] = xi
        J = np.zeros(9)
        det = lib().orc_jacobian(self.h, e, _p(xi3), _p(J))
        return det, J.reshape(3, 3)


# standalone graph algorithms
def graph_tarjan(nv, edges):
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    comp = np.zeros(nv, np.int32)
    n = lib().orc_graph_tarjan(nv, e.shape[0], _p(e), _p(comp))
    sccs = [[] for _ in range(n)]
    for v in range(nv):
        sccs[comp[v]].append(v)
    return sccs


def graph_order(nv, edges, weights, mode, threshold=10):
    """mode 0 exact FAS, 1 heuristic FAS, 2 sweep_ordering."""
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    w = np.ascontiguousarray(np.asarray(weights, np.float64))
    order = np.zeros(nv, np.int32)
    nl = np.zeros(1, np.int32)
    lag = np.zeros(max(len(w), 1), np.int32)
    tw = lib().orc_graph_order(nv, e.shape[0], _p(e), _p(w), mode, threshold, _p(order), _p(nl), _p(lag))
    return list(order), list(lag[: nl[0]]), tw


def gauss_legendre(n):
    p = np.zeros(n)
    w = np.zeros(n)
    lib().orc_gauss_legendre(n, _p(p), _p(w))
    return p, w


def gauss_lobatto(n):
    p = np.zeros(n)
    lib().orc_gauss_lobatto(n, _p(p))
    return p


def basis_eval(dim, order, xi):
    nb = (order + 1) ** dim
    xi3 = np.zeros(3)
    xi3[: len(xi)] = xi
    v = np.zeros(nb)
    g = np.zeros(nb * dim)
    lib().orc_basis_eval(dim, order, _p(xi3), _p(v), _p(g))
    return v, g.reshape(nb, dim)
