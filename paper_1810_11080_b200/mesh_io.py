"""JSON mesh files (mesh_io.hpp:14-78): read / write the reference's mesh format.

Format (mesh_io.hpp:14-27)::

    {"order": r, "dim": 2,
     "control_points": [[x, y], ...],
     "elements": [{"nodes": [...], "region": id}, ...],
     "boundary": [{"elem": e, "face": f, "attr": a}, ...]}

``nodes`` are the (r+1)^dim control points of an element in lexicographic order
(x fastest), ``face`` the local face number (mesh.hpp:64-109).  The reference
reads ``dim = 2`` only (mesh_io.hpp:34); this reader also accepts ``dim = 3``
(hexahedra, 6 local faces, ``[x, y, z]`` points) for the 3D generalisation.

Errors mirror the reference's ``MeshError`` messages (mesh_io.hpp:31-61); the
geometric validation that ``HighOrderMesh::build`` performs (face pairing,
Jacobians) runs when the mesh reaches ``hsw_create`` (``SweepSolver``).
"""
from __future__ import annotations

import dataclasses
import json
from typing import Dict, Optional, Tuple

import numpy as np

from .problem import Problem
from .solver import MeshError

__all__ = ["Mesh", "mesh_to_json", "mesh_from_json", "read_mesh", "write_mesh", "mesh_of", "problem_from_mesh"]


@dataclasses.dataclass
class Mesh:
    """The mesh part of a :class:`Problem` (HighOrderMesh's inputs, mesh.hpp:121-134)."""

    dim: int
    order: int
    points: np.ndarray          # (P, dim) float64
    element_nodes: np.ndarray   # (E, (order+1)^dim) int32
    element_region: np.ndarray  # (E,) int32
    bfaces: np.ndarray          # (B, 3) int32: elem, local face, attr


def mesh_of(problem: Problem) -> Mesh:
    return Mesh(problem.dim, problem.geom_order, problem.points, problem.element_nodes,
                problem.element_region, problem.bfaces)


def mesh_to_json(mesh) -> dict:
    """mesh_io.hpp:14-27 (also accepts a Problem)."""
    if isinstance(mesh, Problem):
        mesh = mesh_of(mesh)
    return {
        "order": int(mesh.order),
        "dim": int(mesh.dim),
        "control_points": [[float(c) for c in p] for p in np.asarray(mesh.points)],
        "elements": [{"nodes": [int(n) for n in nodes], "region": int(r)}
                     for nodes, r in zip(np.asarray(mesh.element_nodes), np.asarray(mesh.element_region))],
        "boundary": [{"elem": int(e), "face": int(f), "attr": int(a)} for e, f, a in np.asarray(mesh.bfaces)],
    }


def mesh_from_json(j) -> Mesh:
    """mesh_io.hpp:29-61: key checks, then points / elements / boundary records."""
    if not isinstance(j, dict):
        raise MeshError("mesh file: expected a JSON object")
    for key in ("order", "dim", "control_points", "elements", "boundary"):
        if key not in j:
            raise MeshError(f"mesh file: missing key '{key}'")
    dim = int(j["dim"])
    if dim not in (2, 3):
        raise MeshError("mesh file: only dim = 2 (reference) or dim = 3 (hexahedra) is supported")
    order = int(j["order"])
    if order < 1:
        raise MeshError("mesh file: order must be >= 1")
    pts = []
    for p in j["control_points"]:
        if not isinstance(p, (list, tuple)) or len(p) != dim:
            what = "an [x, y] pair" if dim == 2 else "an [x, y, z] triple"
            raise MeshError(f"mesh file: control point {len(pts)} is not {what}")
        pts.append([float(c) for c in p])
    npe = (order + 1) ** dim
    nodes, region = [], []
    for i, e in enumerate(j["elements"]):
        if "nodes" not in e:
            raise MeshError(f"mesh file: element {i} has no 'nodes'")
        nd = [int(n) for n in e["nodes"]]
        if len(nd) != npe:   # HighOrderMesh::build's node-count invariant (mesh.hpp:121-134)
            raise MeshError(f"mesh: element {i} has {len(nd)} nodes, expected {npe}")
        if any(n < 0 or n >= len(pts) for n in nd):
            raise MeshError(f"mesh: element {i} references a control point out of range")
        nodes.append(nd)
        region.append(int(e.get("region", 1)))
    nfaces = 2 * dim
    bf = []
    for b in j["boundary"]:
        if "elem" not in b or "face" not in b:
            raise MeshError("mesh file: boundary record needs 'elem' and 'face'")
        e, f = int(b["elem"]), int(b["face"])
        if not (0 <= e < len(nodes)) or not (0 <= f < nfaces):
            raise MeshError(f"mesh: boundary face ({e}, {f}) out of range")
        bf.append([e, f, int(b.get("attr", 1))])
    return Mesh(dim, order, np.asarray(pts, np.float64).reshape(-1, dim),
                np.asarray(nodes, np.int32).reshape(-1, npe), np.asarray(region, np.int32),
                np.asarray(bf, np.int32).reshape(-1, 3))


def write_mesh(mesh, path: str) -> None:
    """mesh_io.hpp:63-67."""
    try:
        with open(path, "w") as fh:
            json.dump(mesh_to_json(mesh), fh, indent=1)
            fh.write("\n")
    except OSError as ex:
        raise MeshError(f"mesh file: cannot open '{path}' for writing") from ex


def read_mesh(path: str) -> Mesh:
    """mesh_io.hpp:69-78."""
    try:
        fh = open(path)
    except OSError as ex:
        raise MeshError(f"mesh file: cannot open '{path}'") from ex
    with fh:
        try:
            j = json.load(fh)
        except json.JSONDecodeError as ex:
            raise MeshError(f"mesh file '{path}': {ex}") from ex
    return mesh_from_json(j)


def problem_from_mesh(mesh: Mesh, ord_weight: np.ndarray, ord_dir: np.ndarray,
                      xs: Dict[int, Tuple[float, float]], basis_order: Optional[int] = None,
                      **kw) -> Problem:
    """A solvable :class:`Problem` on an ingested mesh: what the reference's
    ``assemble_transport_operator`` is handed after ``read_mesh`` (config.hpp)."""
    return Problem(mesh.dim, mesh.order, basis_order if basis_order is not None else mesh.order,
                   np.asarray(mesh.points, np.float64), np.asarray(mesh.element_nodes, np.int32),
                   np.asarray(mesh.element_region, np.int32), np.asarray(mesh.bfaces, np.int32),
                   np.asarray(ord_weight, np.float64), np.asarray(ord_dir, np.float64), dict(xs), **kw)
