"""Synthetic meshes for the BASELINE.json configurations (host plumbing).

The reference only ships a spider-web tube and a voxel bifurcation
(/root/reference/proj/src/mesh_gen.cpp:108-279); the BASELINE configs name a
hex-grid-mapped cylinder (configs 0/1) and Delaunay meshes (2-4), which are
new generators.  Meshes are fed to the reference
through the same arrays (oracle harness) so both sides see identical inputs.
"""
from __future__ import annotations

import itertools

import numpy as np

from .mesh import DIRICHLET, NEUMANN, Mesh, Patch, boundary_faces

# Kuhn (Freudenthal) split: one tet per axis permutation, all sharing the
# hex main diagonal, so neighbouring hexes split shared faces identically.
_KUHN = [
    [0, a, a + b, 7]
    for (a, b) in (
        (1 << p[0], 1 << p[1]) for p in itertools.permutations((0, 1, 2))
    )
]


def hex_cylinder(radius: float, length: float, nx: int, ny: int, nz: int) -> Mesh:
    """nx x ny x nz hex grid on [-1,1]^2 x [0,L], square mapped to the disk of
    `radius` (elliptical map), 6 Kuhn tets per hex.  Patches: `inlet` (z=0,
    Dirichlet), `outlet` (z=L, Neumann), `wall` (Dirichlet).  Config 0 is
    (0.3, 6, 10, 10, 60) -> 36,000 tets / 7,381 nodes; config 1 is
    (0.3, 6, 20, 20, 120) -> 288,000 tets / 53,361 nodes."""
    s = -1.0 + 2.0 * np.arange(nx + 1) / nx
    t = -1.0 + 2.0 * np.arange(ny + 1) / ny
    z = length * np.arange(nz + 1) / nz
    S, T = np.meshgrid(s, t, indexing="xy")  # (ny+1, nx+1)
    X = radius * S * np.sqrt(1.0 - 0.5 * T * T)
    Y = radius * T * np.sqrt(1.0 - 0.5 * S * S)
    nxy = (nx + 1) * (ny + 1)
    xyz = np.empty(((nz + 1) * nxy, 3))
    for k in range(nz + 1):
        xyz[k * nxy:(k + 1) * nxy, 0] = X.reshape(-1)
        xyz[k * nxy:(k + 1) * nxy, 1] = Y.reshape(-1)
        xyz[k * nxy:(k + 1) * nxy, 2] = z[k]

    kk, jj, ii = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    base = (kk * (ny + 1) + jj) * (nx + 1) + ii  # (nz,ny,nx), hex-major order
    base = base.reshape(-1)
    corner = np.array(
        [
            (dz * (ny + 1) + dy) * (nx + 1) + dx
            for c in range(8)
            for dx, dy, dz in [((c >> 0) & 1, (c >> 1) & 1, (c >> 2) & 1)]
        ]
    )
    hexv = base[:, None] + corner[None, :]  # (nhex, 8), corner bit0=x bit1=y bit2=z
    conn = hexv[:, np.array(_KUHN)].reshape(-1, 4).astype(np.int32)

    bf = boundary_faces(conn, xyz.shape[0])
    zc = xyz[bf, 2].mean(axis=1)
    tol = 1e-9 * length
    inlet = bf[zc < tol]
    outlet = bf[zc > length - tol]
    wall = bf[(zc >= tol) & (zc <= length - tol)]
    mesh = Mesh(
        xyz=xyz,
        conn=conn,
        patches=[
            Patch("inlet", DIRICHLET, inlet),
            Patch("outlet", NEUMANN, outlet),
            Patch("wall", DIRICHLET, wall),
        ],
    )
    return mesh.finalize()


def _morton(p: np.ndarray, bits: int = 16) -> np.ndarray:
    """Morton (Z-order) key of points in their bounding box."""
    lo, hi = p.min(axis=0), p.max(axis=0)
    q = ((p - lo) / np.maximum(hi - lo, 1e-300) * ((1 << bits) - 1)).astype(np.uint64)
    key = np.zeros(len(p), dtype=np.uint64)
    for b in range(bits):
        for d in range(3):
            key |= ((q[:, d] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + d)
    return key


def cube_delaunay(npoints: int, seed: int = 4) -> Mesh:
    """BASELINE config 4: Delaunay tetrahedralisation (scipy / Qhull) of
    `npoints` seeded uniform points in the unit cube.  Nodes and elements are
    renumbered along a Morton curve (the GPU kernels' gathers and element
    chunks rely on spatial locality of the numbering).  Boundary facets are
    split by outward normal: `inlet` (n_x <= -0.8, Dirichlet), `outlet`
    (n_x >= 0.8, Neumann), `wall` (the rest, Dirichlet)."""
    from scipy.spatial import Delaunay

    pts = np.random.default_rng(seed).random((npoints, 3))
    perm = np.argsort(_morton(pts), kind="stable")
    pts = pts[perm]
    tri = Delaunay(pts)
    conn = tri.simplices.astype(np.int32)
    conn = conn[np.argsort(_morton(pts[conn].mean(axis=1)), kind="stable")]
    mesh = Mesh(xyz=pts, conn=conn, patches=[])
    mesh.finalize()  # orientation only (no patches yet)
    bf = boundary_faces(mesh.conn, mesh.num_nodes)
    a, b, c = pts[bf[:, 0]], pts[bf[:, 1]], pts[bf[:, 2]]
    nrm = np.cross(b - a, c - a)
    nrm /= np.linalg.norm(nrm, axis=1)[:, None]
    # orient outward: away from the cube centre (the hull is convex)
    flip = np.einsum("ij,ij->i", nrm, (a + b + c) / 3.0 - 0.5) < 0
    nrm[flip] = -nrm[flip]
    inlet = nrm[:, 0] <= -0.8
    outlet = nrm[:, 0] >= 0.8
    mesh.patches = [
        Patch("inlet", DIRICHLET, bf[inlet]),
        Patch("outlet", NEUMANN, bf[outlet]),
        Patch("wall", DIRICHLET, bf[~inlet & ~outlet]),
    ]
    return mesh.finalize()


def config_mesh(cfg: int) -> Mesh:
    if cfg == 0:
        return hex_cylinder(0.3, 6.0, 10, 10, 60)
    if cfg == 1:
        return hex_cylinder(0.3, 6.0, 20, 20, 120)
    if cfg == 4:
        return cube_delaunay(700_000, seed=4)
    raise ValueError(f"no generator for config {cfg} yet")
