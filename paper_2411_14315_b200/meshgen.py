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


def _disk_map(S: np.ndarray, T: np.ndarray):
    """Elliptical square -> unit disk map used by every swept tube."""
    return S * np.sqrt(1.0 - 0.5 * T * T), T * np.sqrt(1.0 - 0.5 * S * S)


def stenosis_tube(nx: int, nz: int, arc_radius: float = 5.0, length: float = 8.0,
                  r_in: float = 0.2, r_out: float = 0.15, area_reduction: float = 0.6,
                  sigma: float = 0.4) -> Mesh:
    """BASELINE config 3 geometry: a vessel swept along a circular centreline
    (radius `arc_radius`, arc length `length`, in the x-z plane), radius
    tapering linearly r_in -> r_out, with a Gaussian constriction of
    `area_reduction` at mid-length:
        r(s) = (r_in + (r_out - r_in) s/L) (1 - d exp(-(s - L/2)^2 / (2 sigma^2))),
        (1 - d)^2 = 1 - area_reduction.
    Structured: nx x nx square cross-sections mapped to the disk, nz slices,
    6 Kuhn tets per hex (consistent diagonals), so the mesh is conforming.
    Patches `inlet` (s=0, Dirichlet), `outlet` (s=L, Neumann), `wall`.
    ~2M tets at (24, 580)."""
    d = 1.0 - np.sqrt(1.0 - area_reduction)
    sv = length * np.arange(nz + 1) / nz
    rad = (r_in + (r_out - r_in) * sv / length) * (1.0 - d * np.exp(-((sv - 0.5 * length) ** 2) / (2 * sigma**2)))
    th = sv / arc_radius
    cen = np.stack([arc_radius * (1.0 - np.cos(th)), np.zeros_like(th), arc_radius * np.sin(th)], axis=1)
    e1 = np.stack([np.cos(th), np.zeros_like(th), -np.sin(th)], axis=1)  # in-plane normal
    e2 = np.array([0.0, 1.0, 0.0])
    g = -1.0 + 2.0 * np.arange(nx + 1) / nx
    S, T = np.meshgrid(g, g, indexing="xy")
    X, Y = _disk_map(S, T)
    X, Y = X.reshape(-1), Y.reshape(-1)
    nxy = (nx + 1) ** 2
    xyz = (cen[:, None, :] + rad[:, None, None] * (X[None, :, None] * e1[:, None, :]
                                                     + Y[None, :, None] * e2[None, None, :]))
    xyz = xyz.reshape(-1, 3)
    kk, jj, ii = np.meshgrid(np.arange(nz), np.arange(nx), np.arange(nx), indexing="ij")
    base = ((kk * (nx + 1) + jj) * (nx + 1) + ii).reshape(-1)
    corner = np.array([(((c >> 2) & 1) * (nx + 1) + ((c >> 1) & 1)) * (nx + 1) + (c & 1) for c in range(8)])
    conn = (base[:, None] + corner[None, :])[:, np.array(_KUHN)].reshape(-1, 4).astype(np.int32)
    bf = boundary_faces(conn, xyz.shape[0])
    sl = (bf // nxy).astype(np.int64)  # slice index of each facet vertex
    inlet = np.all(sl == 0, axis=1)
    outlet = np.all(sl == nz, axis=1)
    mesh = Mesh(xyz=xyz, conn=conn, patches=[
        Patch("inlet", DIRICHLET, bf[inlet]),
        Patch("outlet", NEUMANN, bf[outlet]),
        Patch("wall", DIRICHLET, bf[~inlet & ~outlet]),
    ])
    return mesh.finalize()


def _tjunction_inside(p: np.ndarray, R: float, r: float, half: float, arm: float, eps: float = 0.0):
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    main = (y * y + z * z < (R - eps) ** 2) & (np.abs(x) < half - eps)
    arms = (x * x + z * z < (r - eps) ** 2) & (np.abs(y) < arm - eps)
    return main | arms


def tjunction_delaunay(npoints: int, seed: int = 2, R: float = 0.6, r: float = 0.5,
                       main_length: float = 10.0, inlet_length: float = 4.0) -> Mesh:
    """BASELINE config 2 geometry: a main tube (radius R, length main_length,
    axis x, two zero-traction outlets at x = +-L/2) joined at x = 0 by two
    inlet tubes (radius r, length inlet_length beyond the main wall, axes +y
    and -y).  Unstructured: seeded points (uniform in the volume plus a
    matching density on every surface), Qhull Delaunay, tets whose centroid is
    outside the union removed, unused points dropped, Morton renumbering.
    Patches: `inlet1` (y = +arm), `inlet2` (y = -arm) Dirichlet, `outlet1`
    (x = -L/2), `outlet2` (x = +L/2) Neumann, `wall` Dirichlet.
    ~1M tets at npoints = 150_000."""
    from scipy.spatial import Delaunay

    rng = np.random.default_rng(seed)
    half, arm = 0.5 * main_length, R + inlet_length
    vol = np.pi * R * R * main_length + 2 * np.pi * r * r * inlet_length
    area = (2 * np.pi * R * main_length + 2 * 2 * np.pi * r * inlet_length
            + 2 * np.pi * R * R + 2 * np.pi * r * r)
    h = (vol / npoints) ** (1.0 / 3.0)
    nsurf = int(area / (h * h))
    nvol = max(npoints - nsurf, 1000)
    box_lo = np.array([-half, -arm, -R])
    box_hi = np.array([half, arm, R])
    pts = []
    need = nvol
    while need > 0:
        c = box_lo + (box_hi - box_lo) * rng.random((2 * need + 1000, 3))
        c = c[_tjunction_inside(c, R, r, half, arm, eps=0.25 * h)]
        pts.append(c[:need])
        need -= len(pts[-1])
    # surface samples: lateral walls (outside the other tube), end caps
    def lateral(n, rad, lo, hi, axis):
        t = rng.uniform(lo, hi, n)
        ph = rng.uniform(0, 2 * np.pi, n)
        a, b = rad * np.cos(ph), rad * np.sin(ph)
        q = np.zeros((n, 3))
        if axis == 0:
            q[:, 0], q[:, 1], q[:, 2] = t, a, b
        else:
            q[:, 1], q[:, 0], q[:, 2] = t, a, b
        return q

    def cap(n, rad, pos, axis):
        rr = rad * np.sqrt(rng.random(n))
        ph = rng.uniform(0, 2 * np.pi, n)
        q = np.zeros((n, 3))
        if axis == 0:
            q[:, 0], q[:, 1], q[:, 2] = pos, rr * np.cos(ph), rr * np.sin(ph)
        else:
            q[:, 1], q[:, 0], q[:, 2] = pos, rr * np.cos(ph), rr * np.sin(ph)
        return q

    dens = 1.0 / (h * h)
    mw = lateral(int(dens * 2 * np.pi * R * main_length), R, -half, half, 0)
    mw = mw[~(mw[:, 0] ** 2 + mw[:, 2] ** 2 < r * r)]  # openings of the inlet tubes
    aw = np.concatenate([lateral(int(dens * 2 * np.pi * r * inlet_length), r, R * s0, arm * s0, 1)
                         if s0 > 0 else lateral(int(dens * 2 * np.pi * r * inlet_length), r, -arm, -R, 1)
                         for s0 in (1.0, -1.0)])
    aw = aw[~(aw[:, 1] ** 2 + aw[:, 2] ** 2 < R * R)]
    caps = np.concatenate([cap(int(dens * np.pi * R * R), R, -half, 0), cap(int(dens * np.pi * R * R), R, half, 0),
                           cap(int(dens * np.pi * r * r), r, arm, 1), cap(int(dens * np.pi * r * r), r, -arm, 1)])
    P = np.concatenate(pts + [mw, aw, caps])
    tri = Delaunay(P)
    conn = tri.simplices.astype(np.int64)
    cen = P[conn].mean(axis=1)
    keep = _tjunction_inside(cen, R, r, half, arm)
    x0, x1, x2, x3 = (P[conn[:, k]] for k in range(4))
    vol6 = np.abs(np.einsum("ij,ij->i", x1 - x0, np.cross(x2 - x0, x3 - x0)))
    keep &= vol6 > 1e-12 * h ** 3
    conn = conn[keep]
    used = np.unique(conn)
    remap = -np.ones(len(P), np.int64)
    remap[used] = np.arange(len(used))
    P = P[used]
    conn = remap[conn]
    perm = np.argsort(_morton(P), kind="stable")
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    P = P[perm]
    conn = inv[conn].astype(np.int32)
    conn = conn[np.argsort(_morton(P[conn].mean(axis=1)), kind="stable")]
    mesh = Mesh(xyz=P, conn=conn, patches=[])
    mesh.finalize()
    bf = boundary_faces(mesh.conn, mesh.num_nodes)
    fc = P[bf].mean(axis=1)
    tol = 1e-9 * main_length
    in1 = np.all(np.abs(P[bf][:, :, 1] - arm) < tol, axis=1)
    in2 = np.all(np.abs(P[bf][:, :, 1] + arm) < tol, axis=1)
    out1 = np.all(np.abs(P[bf][:, :, 0] + half) < tol, axis=1)
    out2 = np.all(np.abs(P[bf][:, :, 0] - half) < tol, axis=1)
    wall = ~(in1 | in2 | out1 | out2)
    del fc
    mesh.patches = [
        Patch("inlet1", DIRICHLET, bf[in1]),
        Patch("inlet2", DIRICHLET, bf[in2]),
        Patch("outlet1", NEUMANN, bf[out1]),
        Patch("outlet2", NEUMANN, bf[out2]),
        Patch("wall", DIRICHLET, bf[wall]),
    ]
    return mesh.finalize()


def config_mesh(cfg: int) -> Mesh:
    if cfg == 0:
        return hex_cylinder(0.3, 6.0, 10, 10, 60)
    if cfg == 1:
        return hex_cylinder(0.3, 6.0, 20, 20, 120)
    if cfg == 2:
        return tjunction_delaunay(150_000, seed=2)
    if cfg == 3:
        return stenosis_tube(24, 580)
    if cfg == 4:
        return cube_delaunay(700_000, seed=4)
    raise ValueError(f"no generator for config {cfg}")
