"""Host plumbing: synthetic meshes, Mesh::finalize semantics, boundary data.
CPU only; compared with the compiled reference where it is present."""
import os

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2411_14315_b200 import cases, meshgen
from paper_2411_14315_b200.mesh import GeometryError, Mesh, Patch

HAVE_REF = os.path.exists(ob.REF_SO)
ref = pytest.mark.skipif(not HAVE_REF, reason="compiled reference absent")


def test_config_mesh_sizes():
    m0 = meshgen.config_mesh(0)
    assert (m0.num_elements, m0.num_nodes) == (36000, 7381)
    assert [p.name for p in m0.patches] == ["inlet", "outlet", "wall"]
    assert [len(p.facets) for p in m0.patches] == [200, 200, 4800]
    # all elements positively oriented, disk cross-section area ~ pi r^2
    g = ob.restated_geometry(m0.xyz, m0.conn)
    assert (g[:, 12] > 0).all()
    assert abs(m0.patches[0].area - np.pi * 0.09) / (np.pi * 0.09) < 0.01


def scrambled(mesh, seed):
    rng = np.random.default_rng(seed)
    conn = mesh.conn.copy()
    flip = rng.random(len(conn)) < 0.5
    conn[flip, 1], conn[flip, 2] = conn[flip, 2].copy(), conn[flip, 1].copy()
    patches = []
    for p in mesh.patches:
        f = p.facets.copy()
        fl = rng.random(len(f)) < 0.5
        f[fl, 1], f[fl, 2] = f[fl, 2].copy(), f[fl, 1].copy()
        patches.append(Patch(p.name, p.kind, f))
    return Mesh(mesh.xyz.copy(), conn, patches)


@ref
def test_finalize_matches_reference():
    base = meshgen.hex_cylinder(0.3, 1.0, 4, 4, 6)
    raw = scrambled(base, 3)
    mine = Mesh(raw.xyz, raw.conn.copy(), [Patch(p.name, p.kind, p.facets.copy()) for p in raw.patches]).finalize()
    theirs = ob.RefMesh.from_mesh(raw).to_mesh()
    assert np.array_equal(mine.conn, theirs.conn)
    assert np.array_equal(mine.dirichlet, theirs.dirichlet)
    for a, b in zip(mine.patches, theirs.patches):
        assert np.array_equal(a.facets, b.facets)
        assert np.allclose(a.normals, b.normals, rtol=0, atol=1e-15)
        assert np.allclose(a.areas, b.areas, rtol=1e-15, atol=0)
    assert abs(mine.characteristic_length() - ob.RefMesh.from_mesh(raw).characteristic_length()) < 1e-15


def test_finalize_rejects_bad_input():
    base = meshgen.hex_cylinder(0.3, 1.0, 2, 2, 2)
    with pytest.raises(GeometryError):
        Mesh(base.xyz, base.conn, base.patches[:2]).finalize()  # boundary not covered
    bad = base.conn.copy()
    bad[0] = [0, 0, 1, 2]
    with pytest.raises(GeometryError):
        Mesh(base.xyz, bad, []).finalize()


def test_parabolic_inflow_carries_the_flow():
    mesh = meshgen.hex_cylinder(0.3, 2.0, 8, 8, 4)
    q = cases.flow_samples(2.0, [0.2, -0.1], [0.05, 0.1], 3, 1.0)
    g = cases.parabolic_dirichlet(mesh, 0, q).reshape(mesh.num_nodes, 3, -1)
    p = mesh.patches[0]
    tri = np.array([[2 / 3, 1 / 6, 1 / 6], [1 / 6, 2 / 3, 1 / 6], [1 / 6, 1 / 6, 2 / 3]])
    gq = np.einsum("qa,faik->fqik", tri, g[p.facets])
    flow = -(p.areas[:, None] / 3 * np.einsum("fqik,fi->fqk", gq, p.normals).sum(1)).sum(0)
    assert np.allclose(flow, q, rtol=1e-12)
    wall = mesh.patches[2].facets.reshape(-1)
    assert np.all(g[wall] == 0.0)


@ref
def test_initial_state_and_pseudo_dt_match_reference():
    import bench

    prob = cases.config_problem(0)
    rc = ob.ref_context(prob)
    s0 = cases.initial_state(prob)
    rs = rc.install_dirichlet(np.zeros_like(s0))
    p0 = rc.initial_pressure()
    rs.reshape(prob.mesh.num_nodes, 4, prob.N)[:, 3, :] = p0 if p0 != 0 else 0.0
    assert np.array_equal(rs, s0)
    assert abs(bench.auto_pseudo_dt(prob) - rc.suggest_pseudo_dt()) < 1e-14 * rc.suggest_pseudo_dt()


def test_random_modes_state_is_real_and_band_limited():
    v = cases.random_modes_state(5, 4, 0).reshape(20, 7)
    c = np.fft.fft(v, axis=1) / 7
    assert np.allclose(c.imag[:, 0], 0, atol=1e-14)
    # |c_k| ~ 1/k^2 scaling: modes 1..3 present, no content beyond M-1
    assert v.shape == (20, 7)


@pytest.mark.parametrize("cfg", [2, 3])
def test_config2_3_generators(cfg):
    """Small instances of the T-junction (Delaunay) and curved stenosis
    (swept, Kuhn) generators: positive volumes, every boundary facet in a
    patch, inflow carried by the inlets, and — when the compiled reference is
    present — Mesh::finalize agreement and residual parity of the restated
    oracle against the reference on the config's boundary data."""
    mesh = meshgen.tjunction_delaunay(3000, seed=2) if cfg == 2 else meshgen.stenosis_tube(4, 24)
    g = ob.restated_geometry(mesh.xyz, mesh.conn)
    assert (g[:, 12] > 0).all()
    names = [p.name for p in mesh.patches]
    if cfg == 2:
        assert names == ["inlet1", "inlet2", "outlet1", "outlet2", "wall"]
    else:
        assert names == ["inlet", "outlet", "wall"]
        # 60 % area stenosis at mid-length: the narrowest slice radius
        nxy = 25
        rad = np.linalg.norm(mesh.xyz[:, 1:2], axis=1).reshape(-1, nxy).max(axis=1)
        assert abs((rad.min() / 0.175) ** 2 - 0.4) < 0.05
    prob = cases.config_problem(cfg, modes=2, mesh=mesh)
    inlets = [k for k, p in enumerate(mesh.patches) if p.name.startswith("inlet")]
    N = prob.N
    gg = prob.dirichlet_g.reshape(mesh.num_nodes, 3, N)
    for k in inlets:
        p = mesh.patches[k]
        tri = np.array([[2 / 3, 1 / 6, 1 / 6], [1 / 6, 2 / 3, 1 / 6], [1 / 6, 1 / 6, 2 / 3]])
        un = np.einsum("fvin,fi->fvn", gg[p.facets], -p.normals)  # inflow through the patch
        flux = (p.areas[:, None] / 3.0 * np.einsum("qv,fvn->fqn", tri, un).sum(axis=1)).sum(axis=0)
        assert (flux > 0).all()
    if HAVE_REF:
        theirs = ob.RefMesh.from_mesh(mesh).to_mesh()
        assert np.array_equal(mesh.conn, theirs.conn)
        s = cases.random_state(mesh.num_nodes, N, 9)
        r_ref = ob.ref_context(prob).residual(s)
        r_orc = ob.Restated(prob).residual(s)
        assert np.linalg.norm(r_orc - r_ref) <= 1e-12 * np.linalg.norm(r_ref)
