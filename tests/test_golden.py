"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py from
the CPU oracle) and full-size properties.

CPU: the oracle and the host plan reproduce the fixtures bit for bit (oracle
regression pin; graph / cut-set / level work is integer-exact).  GPU: the CUDA
sweep matches the fixtures within the north-star tolerance, and at the full C4
size — where the oracle is minutes per sweep — the sweep map is checked through
properties that need no oracle: it is affine in (phi, psi_old) and bit-wise
deterministic.
"""
import os

import numpy as np
import pytest

from paper_1810_11080_b200 import problem as pb

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
CASES = {
    "c1": dict(),
    "c2": dict(cells=6, n_mu=2, n_az=8),
    "c3": dict(cells=3, n_mu=2, n_az=4),
    "c4": dict(cells=2, n_mu=2, n_az=4),
    "c5": dict(cells=2, n_mu=2, n_az=4),
}
SWEEP_TOL = 1e-10
SI_TOL = 1e-8


def _gold(name):
    return np.load(os.path.join(GOLD, f"{name}_small.npz"))


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_reproduces_golden_bit_for_bit(name):
    import oracle as O
    g = _gold(name)
    prob = pb.config(name, **CASES[name])
    orc = O.OracleSolver(prob)
    assert np.array_equal(orc.sweep_all(g["phi"], g["psi_old"]), g["psi_new"])
    for d in range(prob.num_ordinates):
        o = orc.ordering(d)
        assert np.array_equal(o["order"], g[f"order_{d}"]) and np.array_equal(o["level"], g[f"level_{d}"])
        assert np.array_equal(o["lagged_edges"], g[f"lagged_{d}"])
    if name == "c1":
        si = orc.source_iteration(1e-8, 400, 1)
        assert si["iterations"] == int(g["si_iterations"])
        assert np.array_equal(si["phi"], g["si_phi"]) and np.array_equal(si["psi"], g["si_psi"])


@pytest.mark.parametrize("name", list(CASES))
def test_host_plan_reproduces_golden_orderings(name):
    import paper_1810_11080_b200 as pk
    g = _gold(name)
    prob = pb.config(name, **CASES[name])
    s = pk.SweepSolver(prob, device=-1)
    for d in range(prob.num_ordinates):
        o = s.ordering(d)
        assert np.array_equal(o.order, g[f"order_{d}"]) and np.array_equal(o.level, g[f"level_{d}"])
        assert np.array_equal(o.lagged_edges, g[f"lagged_{d}"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_sweep_matches_golden(name):
    import paper_1810_11080_b200 as pk
    g = _gold(name)
    prob = pb.config(name, **CASES[name])
    s = pk.SweepSolver(prob, pk.SolveOptions(tolerance=1e-8, criterion="phi_rel_l2"))
    assert rel_l2(s.sweep(-1, g["phi"], g["psi_old"]), g["psi_new"]) <= SWEEP_TOL
    for d in range(prob.num_ordinates):
        o = s.ordering(d)
        assert np.array_equal(o.order, g[f"order_{d}"]) and np.array_equal(o.lagged_edges, g[f"lagged_{d}"])
    if name == "c1":
        state, hist = s.source_iteration()
        assert hist.iterations() == int(g["si_iterations"])
        assert rel_l2(state.phi, g["si_phi"]) <= SI_TOL and rel_l2(state.psi, g["si_psi"]) <= SI_TOL


class _DevView:
    """Raw device pointer as a torch-importable array (__cuda_array_interface__)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


@pytest.mark.gpu
def test_full_c4_sweep_is_affine_and_deterministic():
    """Full C4 (8.4 M local solves per sweep), device-resident: S(phi, psi_old)
    is affine, so S((x + y) / 2) = (S(x) + S(y)) / 2 up to rounding, and two
    identical sweeps agree bit for bit (no atomics or order dependence)."""
    import ctypes as C
    import torch
    import paper_1810_11080_b200 as pk
    from paper_1810_11080_b200 import _capi
    prob = pb.config("c4")
    s = pk.SweepSolver(prob)
    L = _capi.load()
    N, nd = prob.num_dofs, prob.num_ordinates
    pa, pb_, ph = C.c_void_p(), C.c_void_p(), C.c_void_p()
    assert L.hsw_device_state(s.handle, C.byref(pa), C.byref(pb_), C.byref(ph)) == 0
    dev = torch.device("cuda", 0)
    psi_a = torch.as_tensor(_DevView(pa.value, (nd, N)), device=dev)
    psi_b = torch.as_tensor(_DevView(pb_.value, (nd, N)), device=dev)
    phi = torch.as_tensor(_DevView(ph.value, (N,)), device=dev)
    g = torch.Generator(device=dev).manual_seed(4)
    x_phi, y_phi = torch.rand(N, generator=g, device=dev, dtype=torch.float64), \
        torch.rand(N, generator=g, device=dev, dtype=torch.float64)
    x_psi = torch.rand((nd, N), generator=g, device=dev, dtype=torch.float64) * 1.5 - 0.5
    y_psi = torch.rand((nd, N), generator=g, device=dev, dtype=torch.float64) * 1.5 - 0.5

    def sweep(ph_in, psi_in):
        phi.copy_(ph_in)
        psi_a.copy_(psi_in)
        torch.cuda.synchronize()
        assert L.hsw_sweep_resident(s.handle) == 0
        assert L.hsw_synchronize(s.handle) == 0, _capi.last_error()
        return psi_b.clone()

    a = sweep(x_phi, x_psi)
    assert torch.equal(sweep(x_phi, x_psi), a)
    b = sweep(y_phi, y_psi)
    x_psi.add_(y_psi).mul_(0.5)
    m = sweep(0.5 * (x_phi + y_phi), x_psi)
    a.add_(b).mul_(0.5)
    err = float(torch.linalg.vector_norm(m - a) / torch.linalg.vector_norm(a))
    assert err <= SWEEP_TOL, err
