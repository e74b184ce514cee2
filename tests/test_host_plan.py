"""Product host logic on CPU (no GPU): the C-ABI library builds the same
interior faces, couplings, graph weights, cut sets, orderings and levels as the
oracle, bit for bit; the ABI exports every declared symbol; error paths map to
the reference's exception types."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import _capi
from paper_1810_11080_b200 import problem as pb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    ("c1", {}),
    ("c1", dict(cells=5)),
    ("c2", dict(cells=24, n_mu=2, n_az=8)),
    ("c3", dict(cells=5, n_mu=2, n_az=6)),
    ("c4", dict(cells=4, n_mu=2, n_az=4)),
    ("c5", dict(cells=3, n_mu=2, n_az=4)),
]


def _compare(prob, weighting="face", thr=10):
    prob = prob.replace(weighting={"unity": 0, "face": 1, "siginvface": 2}[weighting], fas_threshold=thr)
    plan = pk.SweepSolver(prob, pk.SolveOptions(weighting=weighting, exact_fas_threshold=thr), device=-1)
    orc = O.OracleSolver(prob, cache_lu=False, check_rcond=False)
    assert (plan.interior_faces() == orc.interior_faces()).all()
    total = 0
    for d in range(prob.num_ordinates):
        pi, pw = plan.couplings(d)
        oi, ow = orc.couplings(d)
        assert pi.shape == oi.shape and (pi == oi).all(), d
        assert (pw == ow).all(), d  # FP64 weights bit-identical
        po, oo = plan.ordering(d), orc.ordering(d)
        assert (po.order == oo["order"]).all() and (po.position == oo["position"]).all()
        assert (po.lagged_edges == oo["lagged_edges"]).all()
        assert po.lagged_weight == oo["lagged_weight"]
        assert (po.level == oo["level"]).all()
        total += len(po.lagged_edges)
    assert plan.total_lagged_edges() == total == orc.total_lagged_edges()
    return total


@pytest.mark.parametrize("name,kw", CASES, ids=[f"{c[0]}-{i}" for i, c in enumerate(CASES)])
def test_plan_bit_exact_against_oracle(name, kw):
    _compare(pb.config(name, **kw))


@pytest.mark.parametrize("weighting", ["unity", "siginvface"])
def test_plan_other_weightings(weighting):  # sweepgraph.hpp:40,60-72
    _compare(pb.config("c2", cells=12, n_mu=2, n_az=8), weighting=weighting)


def test_plan_exact_fas_threshold_variants():  # mixes DP and heuristic components
    prob = pb.config("c2", cells=20, n_mu=2, n_az=8)
    assert _compare(prob, thr=3) > 0
    _compare(prob, thr=22)


def test_full_c1_and_c2_cut_sets():
    assert _compare(pb.config("c1")) == 48
    _compare(pb.config("c2", cells=64))


def test_abi_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "hosweep_b200.h")).read()
    declared = set(re.findall(r"\b(hsw_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(_capi.EXPORTED), declared ^ set(_capi.EXPORTED)
    lib = C.CDLL(_capi.LIB_PATH)
    for sym in declared:
        assert hasattr(lib, sym), sym


def test_no_device_handle_fails_loudly():
    plan = pk.SweepSolver(pb.config("c1", cells=2), device=-1)
    with pytest.raises(pk.solver.CudaError, match="no CPU fallback"):
        plan.sweep(-1, np.zeros(plan.num_dofs), np.zeros((plan.num_ordinates, plan.num_dofs)))
    with pytest.raises(IndexError):
        plan.ordering(plan.num_ordinates)


def test_mesh_errors_map_to_reference_exceptions():  # mesh.hpp:242-339, xsec.hpp:63-66
    pts, nodes, bf = pb.generate_uniform(2, 2, 1)
    w, d = pb.level_symmetric_2d(2)
    base = pb.Problem(2, 1, 1, pts, nodes, np.ones(4, np.int32), bf, w, d, {1: (1.0, 0.5)})
    with pytest.raises(pk.MeshError, match="neither interior nor declared boundary"):
        pk.SweepSolver(base.replace(bfaces=bf[1:]), device=-1)
    with pytest.raises(pk.MeshError, match="boundary record for interior face"):
        pk.SweepSolver(base.replace(bfaces=np.vstack([bf, [[0, 1, 9]]]).astype(np.int32)), device=-1)
    bad = nodes.copy()
    bad[0] = bad[0][[1, 0, 3, 2]]  # mirrored element: det(J) < 0
    with pytest.raises(pk.MeshError):
        pk.SweepSolver(base.replace(element_nodes=bad), device=-1)
    with pytest.raises(ValueError, match="sigma_t >= sigma_s"):
        pk.SweepSolver(base.replace(xs={1: (1.0, 2.0)}), device=-1)
    with pytest.raises(pk.MeshError, match="out of range"):
        pk.SweepSolver(base.replace(element_nodes=nodes + 100), device=-1)


def test_product_quadrature_and_configs():
    for dim, nmu, naz in [(2, 2, 8), (2, 4, 16), (3, 8, 16), (3, 8, 32)]:
        w, d = pb.product_quadrature(dim, nmu, naz)
        assert len(w) == nmu * naz and abs(w.sum() - 4 * math.pi) < 1e-12
        assert np.abs(np.linalg.norm(d, axis=1) - 1).max() < 1e-14
        assert np.abs(d[:, :2]).min() > 1e-3  # no azimuth exactly along an axis
    c2 = pb.config("c2", cells=16)
    frac10 = np.mean(c2.element_region == 2)
    assert 0.15 < frac10 < 0.45
    c5 = pb.config("c5", cells=10)
    assert set(np.unique(c5.element_region)) == {1, 2, 3}
