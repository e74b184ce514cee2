"""JSON mesh ingest (mesh_io.hpp:14-78): round trip, the reference's error
messages, and a solvable plan from an ingested mesh identical to the original."""
import json

import numpy as np
import pytest

import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import mesh_io as mio
from paper_1810_11080_b200 import problem as pb


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c3", dict(cells=3, n_mu=2, n_az=4))])
def test_round_trip_and_plan(tmp_path, name, kw):
    prob = pb.config(name, **kw)
    path = str(tmp_path / "mesh.json")
    mio.write_mesh(prob, path)
    m = mio.read_mesh(path)
    assert m.dim == prob.dim and m.order == prob.geom_order
    assert np.array_equal(m.points, prob.points)          # JSON doubles round-trip exactly (repr)
    assert np.array_equal(m.element_nodes, prob.element_nodes)
    assert np.array_equal(m.element_region, prob.element_region)
    assert np.array_equal(m.bfaces, prob.bfaces)
    p2 = mio.problem_from_mesh(m, prob.ord_weight, prob.ord_dir, prob.xs, basis_order=prob.basis_order,
                               source_kind=prob.source_kind, source_params=prob.source_params)
    a = pk.SweepSolver(prob, device=-1)
    b = pk.SweepSolver(p2, device=-1)
    assert (a.interior_faces() == b.interior_faces()).all()
    for d in range(prob.num_ordinates):
        oa, ob = a.ordering(d), b.ordering(d)
        assert (oa.order == ob.order).all() and (oa.lagged_edges == ob.lagged_edges).all()


def test_reference_error_messages(tmp_path):
    j = mio.mesh_to_json(pb.config("c1", cells=2))
    with pytest.raises(pk.MeshError, match="expected a JSON object"):
        mio.mesh_from_json([1, 2])
    for key in ("order", "dim", "control_points", "elements", "boundary"):
        bad = dict(j)
        del bad[key]
        with pytest.raises(pk.MeshError, match=f"missing key '{key}'"):
            mio.mesh_from_json(bad)
    with pytest.raises(pk.MeshError, match="only dim"):
        mio.mesh_from_json(dict(j, dim=4))
    with pytest.raises(pk.MeshError, match="order must be >= 1"):
        mio.mesh_from_json(dict(j, order=0))
    with pytest.raises(pk.MeshError, match="control point 1 is not an \\[x, y\\] pair"):
        mio.mesh_from_json(dict(j, control_points=[[0.0, 0.0], [1.0]]))
    with pytest.raises(pk.MeshError, match="cannot open"):
        mio.read_mesh(str(tmp_path / "absent.json"))
    p = tmp_path / "broken.json"
    p.write_text("{ not json")
    with pytest.raises(pk.MeshError, match="broken.json"):
        mio.read_mesh(str(p))
    # region / attr defaults (mesh_io.hpp:46,54)
    j2 = json.loads(json.dumps(j))
    for e in j2["elements"]:
        e.pop("region")
    for b in j2["boundary"]:
        b.pop("attr")
    m = mio.mesh_from_json(j2)
    assert (m.element_region == 1).all() and (m.bfaces[:, 2] == 1).all()
