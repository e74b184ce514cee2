"""Problem description and the synthetic inputs of BASELINE.json's configs.

This is input construction on either side of the sweep path: the mesh
generators (restating ``generate_uniform``, generators.hpp:24-67, and its
node-displacement pattern, generators.hpp:184-208, with the configs' twist),
the product angular quadrature the configs need (the reference only has
level-symmetric sets, angular.hpp:39-80), seeded per-element materials and the
volumetric source.  The same :class:`Problem` arrays are handed to the CUDA
solver (``paper_1810_11080_b200.SweepSolver``) and, in tests, to the CPU oracle.

Conventions (SURVEY.md §8d "conventions the builder must fix"):
  * weights: configs normalise to sum 1; internally the reference's 4*pi
    normalisation is used (angular.hpp:22, solver.hpp:108), so
    ``ord_weight = 4*pi*w_hat`` and phi_config = phi / (4*pi).
  * azimuths phi_k = (k + 1/2) * 2*pi / N_az (never exactly along an axis).
  * 2D: "mu > 0" nodes = Gauss-Legendre on (0, 1) for the polar cosine
    (z component); streaming uses the (x, y) components (assembly.hpp:383).
  * 3D: full-sphere Gauss-Legendre on (-1, 1) for the polar cosine.
  * RNG: std::mt19937_64(seed), u = (x >> 11) * 2^-53, drawn in element order.
  * face rule: Gauss-Legendre with p+2 points (FaceIntegration::Rule::gauss).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Optional, Tuple

import numpy as np

__all__ = [
    "Problem", "gauss_lobatto", "generate_uniform", "generate_uniform_3d", "twist_2d",
    "twist_3d", "product_quadrature", "level_symmetric_2d", "MT19937_64", "config",
    "CONFIG_NAMES",
]


@dataclasses.dataclass
class Problem:
    """Everything ``assemble_transport_operator`` (assembly.hpp:362) takes:
    mesh, basis order, ordinates, cross sections, source spec, and the
    ``SolveOptions`` graph knobs (solver.hpp:25-32)."""

    dim: int
    geom_order: int
    basis_order: int
    points: np.ndarray          # (P, dim) float64 control points
    element_nodes: np.ndarray   # (E, (r+1)^dim) int32, lexicographic, x fastest
    element_region: np.ndarray  # (E,) int32 material region ids
    bfaces: np.ndarray          # (B, 3) int32 (elem, local_face, attr)
    ord_weight: np.ndarray      # (N,) float64, sum 4*pi
    ord_dir: np.ndarray         # (N, 3) float64 unit directions
    xs: Dict[int, Tuple[float, float]]  # region -> (sigma_t, sigma_s)
    source_kind: int = 0        # 0 constant q; 1 ball indicator
    source_params: Tuple[float, ...] = (1.0,)
    inflow: float = 0.0         # isotropic incident flux (SourceSpec::isotropic)
    volume_points: int = 0      # 0 -> p + 2 per axis (assembly.hpp:146)
    face_points: int = 0        # 0 -> p + 2 Gauss points per face axis
    face_rule: int = 0          # FaceIntegration::Rule (assembly.hpp:33-40): 0 gauss, 1 romberg (2D)
    romberg_tol: float = 1e-10  # FaceIntegration defaults (assembly.hpp:36-38)
    romberg_max_levels: int = 16
    romberg_min_levels: int = 6
    weighting: int = 1          # 0 unity, 1 face (default), 2 siginvface
    fas_threshold: int = 10     # exact FAS up to this SCC size (solver.hpp:31)
    name: str = "custom"

    @property
    def num_elements(self) -> int:
        return int(self.element_nodes.shape[0])

    @property
    def num_ordinates(self) -> int:
        return int(self.ord_weight.shape[0])

    @property
    def block_size(self) -> int:
        return (self.basis_order + 1) ** self.dim

    @property
    def num_dofs(self) -> int:
        return self.num_elements * self.block_size

    def region_arrays(self):
        ids = sorted(self.xs)
        st = np.array([self.xs[i][0] for i in ids], dtype=np.float64)
        ss = np.array([self.xs[i][1] for i in ids], dtype=np.float64)
        return np.array(ids, dtype=np.int32), st, ss

    def source_param_array(self) -> np.ndarray:
        a = np.zeros(8, dtype=np.float64)
        a[: len(self.source_params)] = self.source_params
        return a

    def replace(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)


# ----------------------------------------------------------------------------
# 1D node sets (quadrature.hpp:23-82), used for node placement only.

def _legendre(n: int, x: float):
    p0, p1 = 1.0, x
    if n == 0:
        return 1.0, 0.0
    for k in range(2, n + 1):
        p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
        p0, p1 = p1, p2
    return p1, n * (x * p1 - p0) / (x * x - 1.0)


def gauss_lobatto(n: int) -> np.ndarray:
    """Gauss-Lobatto points on [0,1], endpoints exactly 0 and 1 (quadrature.hpp:62-82)."""
    if n < 2:
        raise ValueError("gauss_lobatto: need n >= 2")
    pts = np.zeros(n)
    pts[-1] = 1.0
    m = n - 1
    for i in range(1, m):
        x = math.cos(math.pi * i / m)
        for _ in range(100):
            p, dp = _legendre(m, x)
            ddp = (2.0 * x * dp - m * (m + 1) * p) / (1.0 - x * x)
            dx = dp / ddp
            x -= dx
            if abs(dx) < 1e-15:
                break
        pts[m - i] = 0.5 * (x + 1.0)
    return pts


def _axis_coords(n_cells: int, order: int, origin: float, h: float) -> np.ndarray:
    """generators.hpp:34-38: global node I = cell*r + k -> origin + cell*h + gl[k]*h."""
    gl = gauss_lobatto(order + 1)
    out = np.empty(n_cells * order + 1)
    for idx in range(n_cells * order + 1):
        cell = min(idx // order, 0 if idx == 0 else (idx - 1) // order)
        k = idx - cell * order
        out[idx] = origin + cell * h + gl[k] * h
    return out


def generate_uniform(nx: int, ny: int, order: int, rect=(0.0, 0.0, 1.0, 1.0)):
    """Axis-aligned grid of order-r quads (generators.hpp:24-67).

    Returns (points (P,2), element_nodes (E,(r+1)^2), bfaces (B,3)); boundary
    attributes 1 bottom, 2 right, 3 top, 4 left."""
    if nx < 1 or ny < 1 or order < 1:
        raise ValueError("generate_uniform: need nx, ny, order >= 1")
    r = order
    x0, y0, x1, y1 = rect
    xs = _axis_coords(nx, r, x0, (x1 - x0) / nx)
    ys = _axis_coords(ny, r, y0, (y1 - y0) / ny)
    npx = nx * r + 1
    X, Y = np.meshgrid(xs, ys, indexing="xy")
    points = np.stack([X.ravel(), Y.ravel()], axis=1)
    ci, cj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    ci, cj = ci.ravel(), cj.ravel()
    ix, iy = np.meshgrid(np.arange(r + 1), np.arange(r + 1), indexing="xy")
    ix, iy = ix.ravel(), iy.ravel()
    nodes = (cj[:, None] * r + iy[None, :]) * npx + (ci[:, None] * r + ix[None, :])
    b = []
    for c in range(nx):
        b.append((c, 0, 1))
        b.append(((ny - 1) * nx + c, 2, 3))
    for c in range(ny):
        b.append((c * nx + nx - 1, 1, 2))
        b.append((c * nx, 3, 4))
    return points, nodes.astype(np.int32), np.array(b, dtype=np.int32)


def generate_uniform_3d(nx: int, ny: int, nz: int, order: int, box=(0, 0, 0, 1, 1, 1)):
    """3D analogue of generate_uniform: element id (ck*ny + cj)*nx + ci, local
    node (iz*(r+1)+iy)*(r+1)+ix.  Local faces: 0 z=0, 1 y=0,
    2 x=1, 3 y=1, 4 x=0, 5 z=1; boundary attrs 1 y=0, 2 x=1, 3 y=1, 4 x=0,
    5 z=0, 6 z=1."""
    r = order
    x0, y0, z0, x1, y1, z1 = box
    xs = _axis_coords(nx, r, x0, (x1 - x0) / nx)
    ys = _axis_coords(ny, r, y0, (y1 - y0) / ny)
    zs = _axis_coords(nz, r, z0, (z1 - z0) / nz)
    npx, npy = nx * r + 1, ny * r + 1
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    points = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    ck, cj, ci = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ck, cj, ci = ck.ravel(), cj.ravel(), ci.ravel()
    iz, iy, ix = np.meshgrid(np.arange(r + 1), np.arange(r + 1), np.arange(r + 1), indexing="ij")
    iz, iy, ix = iz.ravel(), iy.ravel(), ix.ravel()
    nodes = ((ck[:, None] * r + iz[None, :]) * npy + (cj[:, None] * r + iy[None, :])) * npx + (
        ci[:, None] * r + ix[None, :])
    eid = lambda i, j, k: (k * ny + j) * nx + i  # noqa: E731
    b = []
    for k in range(nz):
        for j in range(ny):
            b.append((eid(0, j, k), 4, 4))
            b.append((eid(nx - 1, j, k), 2, 2))
    for k in range(nz):
        for i in range(nx):
            b.append((eid(i, 0, k), 1, 1))
            b.append((eid(i, ny - 1, k), 3, 3))
    for j in range(ny):
        for i in range(nx):
            b.append((eid(i, j, 0), 0, 5))
            b.append((eid(i, j, nz - 1), 5, 6))
    return points, nodes.astype(np.int32), np.array(b, dtype=np.int32)


def twist_2d(points: np.ndarray, amplitude: float, width: float = 0.3, center=(0.5, 0.5)):
    """Rotate every node about ``center`` by theta(r) = A*exp(-(r/w)^2)."""
    dx = points[:, 0] - center[0]
    dy = points[:, 1] - center[1]
    r = np.sqrt(dx * dx + dy * dy)
    th = amplitude * np.exp(-(r / width) ** 2)
    c, s = np.cos(th), np.sin(th)
    out = points.copy()
    out[:, 0] = center[0] + (c * dx - s * dy)
    out[:, 1] = center[1] + (s * dx + c * dy)
    return out


def twist_3d(points: np.ndarray, amplitude: float, width: float = 0.3, center=(0.5, 0.5)):
    """Rotate about the vertical axis through ``center`` by
    theta = A*exp(-(r/w)^2)*(0.5 + z), r the distance to the axis."""
    dx = points[:, 0] - center[0]
    dy = points[:, 1] - center[1]
    r = np.sqrt(dx * dx + dy * dy)
    th = amplitude * np.exp(-(r / width) ** 2) * (0.5 + points[:, 2])
    c, s = np.cos(th), np.sin(th)
    out = points.copy()
    out[:, 0] = center[0] + (c * dx - s * dy)
    out[:, 1] = center[1] + (s * dx + c * dy)
    return out


# ----------------------------------------------------------------------------
# Angular quadratures

def product_quadrature(dim: int, n_mu: int, n_az: int):
    """Product Gauss-Legendre (polar cosine) x equally spaced azimuths.

    Returns (weights summing to 4*pi, dirs (N,3)).  Ordinate index
    d = i_mu * n_az + k.  2D: polar cosines are GL nodes on (0,1) (upper
    hemisphere; the (x,y) components stream).  3D: GL nodes on (-1,1)."""
    x, w = np.polynomial.legendre.leggauss(n_mu)
    if dim == 2:
        xi = 0.5 * (x + 1.0)
        wmu = 0.5 * w          # sums to 1
    else:
        xi = x
        wmu = 0.5 * w          # sums to 1
    az = (np.arange(n_az) + 0.5) * (2.0 * np.pi / n_az)
    dirs, wts = [], []
    for i in range(n_mu):
        st = math.sqrt(max(0.0, 1.0 - xi[i] * xi[i]))
        for k in range(n_az):
            dirs.append((st * math.cos(az[k]), st * math.sin(az[k]), xi[i]))
            wts.append(wmu[i] / n_az)
    wts = np.array(wts)
    wts = wts / wts.sum()
    return 4.0 * np.pi * wts, np.array(dirs, dtype=np.float64)


def level_symmetric_2d(n: int):
    """angular.hpp:39-80: level-symmetric S2/S4, upper hemisphere, weights 4*pi."""
    four_pi = 4.0 * math.pi
    dirs, wts = [], []
    if n == 2:
        a = math.sqrt(3.0) / 3.0
        for sz in (-1, 1):
            for sy in (-1, 1):
                for sx in (-1, 1):
                    dirs.append((sx * a, sy * a, sz * a))
                    wts.append(four_pi / 8.0)
    elif n == 4:
        mu1 = 0.3500212
        mu2 = math.sqrt(mu1 * mu1 + (1.0 - 3.0 * mu1 * mu1))
        base = [(mu2, mu1, mu1), (mu1, mu2, mu1), (mu1, mu1, mu2)]
        for sz in (-1, 1):
            for sy in (-1, 1):
                for sx in (-1, 1):
                    for b in base:
                        dirs.append((sx * b[0], sy * b[1], sz * b[2]))
                        wts.append(four_pi / 24.0)
    else:
        raise ValueError("level_symmetric: only S_2 and S_4 are supported")
    keep = [i for i, dd in enumerate(dirs) if dd[2] > 0.0]
    return (np.array([2.0 * wts[i] for i in keep]), np.array([dirs[i] for i in keep]))


# ----------------------------------------------------------------------------
class MT19937_64:
    """std::mt19937_64 (seeded like the C++ constructor)."""

    _M64 = (1 << 64) - 1

    def __init__(self, seed: int = 5489):
        self.mt = [0] * 312
        self.mt[0] = seed & self._M64
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & self._M64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def next(self) -> int:
        if self.idx >= 312:
            self._twist()
        x = self.mt[self.idx]
        self.idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & self._M64

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / 9007199254740992.0)


def _materials(n: int, seed: int, cuts, regions):
    rng = MT19937_64(seed)
    out = np.empty(n, dtype=np.int32)
    for e in range(n):
        u = rng.uniform()
        k = 0
        while k < len(cuts) and u >= cuts[k]:
            k += 1
        out[e] = regions[k]
    return out


CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5")
DEFAULT_SEED = 20181026


def config(name: str, cells: Optional[int] = None, n_mu: Optional[int] = None,
           n_az: Optional[int] = None, seed: int = DEFAULT_SEED) -> Problem:
    """BASELINE.json configs[0..4] as synthetic problems.

    ``cells``/``n_mu``/``n_az`` shrink a config (same geometry family, order,
    physics) for parity tests; the defaults are the full configs."""
    name = name.lower()
    if name == "c1":
        # configs[0]: 2D 8x8 Q2, twist 0.5, 2 mu x 8 az, sigma_t=1, sigma_s=0.5, q=1
        n = cells or 8
        pts, nodes, bf = generate_uniform(n, n, 2)
        pts = twist_2d(pts, 0.5)
        w, d = product_quadrature(2, n_mu or 2, n_az or 8)
        return Problem(2, 2, 2, pts, nodes, np.ones(len(nodes), np.int32), bf, w, d,
                       {1: (1.0, 0.5)}, 0, (1.0,), name="c1")
    if name == "c2":
        # configs[1]: 2D 128^2 Q3, twist 1.0, 4 mu x 16 az, sigma_t {10 p=.3, 1}, c=0.9,
        # q=1 in the disc r<0.2
        n = cells or 128
        pts, nodes, bf = generate_uniform(n, n, 3)
        pts = twist_2d(pts, 1.0)
        w, d = product_quadrature(2, n_mu or 4, n_az or 16)
        reg = _materials(len(nodes), seed, [0.3], [2, 1])
        return Problem(2, 3, 3, pts, nodes, reg, bf, w, d,
                       {1: (1.0, 0.9), 2: (10.0, 9.0)}, 1,
                       (0.5, 0.5, 0.0, 0.2, 1.0, 0.0), name="c2")
    if name == "c3":
        # configs[2]: 3D 16^3 Q2, twist 0.8*(0.5+z), 8 mu x 16 az, sigma_t=1, c=0.5, q=1
        n = cells or 16
        pts, nodes, bf = generate_uniform_3d(n, n, n, 2)
        pts = twist_3d(pts, 0.8)
        w, d = product_quadrature(3, n_mu or 8, n_az or 16)
        return Problem(3, 2, 2, pts, nodes, np.ones(len(nodes), np.int32), bf, w, d,
                       {1: (1.0, 0.5)}, 0, (1.0,), name="c3")
    if name == "c4":
        # configs[3]: 3D 32^3 Q3, twist 1.0, 8 mu x 32 az, sigma_t {10 p=.3, 1}, c=0.9,
        # q=1 in the ball r<0.2
        n = cells or 32
        pts, nodes, bf = generate_uniform_3d(n, n, n, 3)
        pts = twist_3d(pts, 1.0)
        w, d = product_quadrature(3, n_mu or 8, n_az or 32)
        reg = _materials(len(nodes), seed, [0.3], [2, 1])
        return Problem(3, 3, 3, pts, nodes, reg, bf, w, d,
                       {1: (1.0, 0.9), 2: (10.0, 9.0)}, 1,
                       (0.5, 0.5, 0.5, 0.2, 1.0, 0.0), name="c4")
    if name == "c5":
        # configs[4]: 3D 24^3 Q4, twist 1.2, 8 mu x 32 az, sigma_t {0.1 .3, 1 .5, 10 .2},
        # c=0.95, q=1 uniform
        n = cells or 24
        pts, nodes, bf = generate_uniform_3d(n, n, n, 4)
        pts = twist_3d(pts, 1.2)
        w, d = product_quadrature(3, n_mu or 8, n_az or 32)
        reg = _materials(len(nodes), seed, [0.3, 0.8], [1, 2, 3])
        return Problem(3, 4, 4, pts, nodes, reg, bf, w, d,
                       {1: (0.1, 0.095), 2: (1.0, 0.95), 3: (10.0, 9.5)}, 0, (1.0,),
                       name="c5")
    raise ValueError(f"unknown config {name!r}")
