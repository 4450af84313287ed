"""Pin the plain-C restatement (oracle/hbgls_oracle.c) against the golden
fixtures produced by the compiled reference, and — where the reference
library is present — against the reference directly on fresh inputs.
CPU only."""
import os

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2411_14315_b200 import cases

from goldens import NAMES, load

HAVE_REF = os.path.exists(ob.REF_SO)


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0))


@pytest.mark.parametrize("name", NAMES)
def test_restatement_matches_golden(name):
    prob, d = load(name)
    orc = ob.Restated(prob, tau_mode=int(d["tau_mode"]), pseudo_dt=d["pseudo_dt_eff"])
    # pattern and geometry: bit-exact (linalg.cpp:10-30, mesh.cpp:159-203)
    assert np.array_equal(orc.row_ptr, d["row_ptr"]) and np.array_equal(orc.col_idx, d["col_idx"])
    assert np.array_equal(ob.restated_geometry(prob.mesh.xyz, prob.mesh.conn), d["geometry"])
    s = d["state"]
    assert rel(orc.residual(s), d["residual"]) < 1e-13
    assert rel(orc.residual(s), d["oracle_residual"]) < 1e-12  # tests/oracles.cpp straight loops
    p = orc.tangent(s)
    assert rel(p, d["pvals"]) < 1e-14
    m = orc.mass()
    assert np.array_equal(m, d["mass"])
    assert rel(orc.matvec(d["pvals"], d["mass"], d["y"]), d["matvec"]) < 1e-13
    inv, deg = orc.jacobi(d["pvals"])
    assert deg == int(d["degenerate"]) and np.array_equal(inv, d["inv_diag"])
    g = orc.gmres(d["pvals"], d["mass"], d["matvec"], d["inv_diag"], restart=40, max_iters=400, tol=1e-9)
    assert g["iterations"] == int(d["gmres_iters"])
    assert rel(g["x"], d["gmres_x"]) < 1e-10


def test_spectral_h_dense_and_fftw_path():
    """H = E^-1 Omega E: restated dense formula vs the reference's dense(),
    its oracle_h_dense, and the FFTW(-shim) apply_many path
    (test_spectral.cpp:104-151 bound 1e-11 omega |v|)."""
    from goldens import GOLDEN

    sp = np.load(os.path.join(GOLDEN, "spectral.npz"))
    for M in (1, 2, 3, 4, 7, 13):
        N = 2 * M - 1
        H = ob.restated_h_dense(M, 0.7)
        assert np.abs(H - sp[f"H_{M}"]).max() <= 1e-12 * max(1.0, np.abs(H).max())
        assert np.abs(H - sp[f"Hora_{M}"]).max() <= 1e-12 * max(1.0, np.abs(H).max())
        v = sp[f"v_{M}"].reshape(-1, N)
        omega = 2 * np.pi / 0.7
        assert np.abs(v @ H.T - sp[f"Hv_{M}"].reshape(-1, N)).max() <= 1e-11 * omega * np.abs(v).max() * N
        assert np.allclose(H, -H.T, atol=1e-12 * omega)  # skew, zero diagonal
        if M == 1:
            assert np.all(H == 0.0)


def test_tangent_is_fd_derivative_of_frozen_residual():
    """P is the exact derivative of the frozen-coefficient residual
    (test_assembly.cpp:340-384), checked on the restatement's tangent."""
    if not HAVE_REF:
        pytest.skip("needs the compiled reference (oracle_frozen_residual)")
    rm = ob.RefMesh.tube(0.5, 1.0, 0.34)
    mesh = rm.to_mesh()
    M, N = 3, 5
    prob = cases.Problem(mesh, M, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 3 * N), [], 0.2)
    ref = ob.ref_context(prob, 0, float("inf"))
    orc = ob.Restated(prob, tau_mode=0)
    s0 = cases.random_state(mesh.num_nodes, N, 5)
    p = orc.tangent(s0)
    dy = cases.random_state(mesh.num_nodes, N, 6)
    free = ~mesh.dirichlet.astype(bool)
    dy.reshape(mesh.num_nodes, 4, N)[~free, :3, :] = 0.0
    h = 1e-6
    fd = (ref.frozen_residual(s0 + h * dy, s0) - ref.frozen_residual(s0 - h * dy, s0)) / (2 * h)
    pd = orc.bsr_matvec(p, dy)
    mask = np.ones((mesh.num_nodes, 4, N), bool)
    mask[~free, :3, :] = False
    mask = mask.reshape(-1)
    assert rel(pd[mask], fd[mask]) < 1e-8


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference absent")
@pytest.mark.parametrize("modes,tau", [(1, 0), (3, 0), (5, 1)])
def test_restatement_matches_reference_fresh(modes, tau):
    prob = cases.config_problem(0, modes=modes)
    ref = ob.ref_context(prob, tau, 0.02)
    orc = ob.Restated(prob, tau_mode=tau, pseudo_dt=0.02)
    s = cases.random_state(prob.mesh.num_nodes, prob.N, 17, 2.0)
    assert rel(orc.residual(s), ref.residual(s, 4)) < 1e-12
    p = orc.tangent(s)
    assert rel(p, ref.tangent(s)) < 1e-14
    y = cases.random_state(prob.mesh.num_nodes, prob.N, 18)
    assert rel(orc.matvec(p, orc.mass(), y), ref.matvec(y, 4)) < 1e-13
    rp, ci = ob.RefMesh.from_mesh(prob.mesh).pattern()
    assert np.array_equal(rp, orc.row_ptr) and np.array_equal(ci, orc.col_idx)


def test_resistance_restatement_is_consistent():
    """The restated resistance outlet (hbgls_oracle.c): its operator part is the
    exact derivative of its residual part (linear in u, Dirichlet columns
    masked), and R = 0 reproduces the plain restatement bit for bit."""
    from oracle.bindings import Restated
    from paper_2411_14315_b200 import cases, meshgen
    from paper_2411_14315_b200.mesh import NEUMANN

    mesh = meshgen.hex_cylinder(0.4, 1.0, 3, 3, 4)
    N = 3
    neu = [(k, np.full(N, -5.0)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    prob = cases.Problem(mesh, 2, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 3 * N), neu, 0.2)
    out = neu[0][0]
    o1, o0 = Restated(prob, resistance={out: 2e4}), Restated(prob)
    oz = Restated(prob, resistance={out: 0.0})
    s = cases.random_state(mesh.num_nodes, N, 5)
    y = cases.random_state(mesh.num_nodes, N, 6)
    assert np.array_equal(oz.residual(s), o0.residual(s))
    p = o0.tangent(s)
    m = o0.mass()
    yf = y.reshape(mesh.num_nodes, 4, N).copy()
    yf[mesh.dirichlet.astype(bool)] = 0.0
    yf = yf.reshape(-1)
    d_r = (o1.residual(s + yf) - o0.residual(s + yf)) - (o1.residual(s) - o0.residual(s))
    d_l = o1.matvec(p, m, y) - o0.matvec(p, m, y)
    assert np.linalg.norm(d_l) > 0
    assert np.linalg.norm(d_r - d_l) <= 1e-10 * np.linalg.norm(d_l)


@pytest.mark.parametrize("name", ["tube_m3_qp", "tube_m4_mean", "bifurcation_m3"])
def test_row_subsets_equal_full_assembly(name):
    """hbo_residual_rows / hbo_tangent_rows (the full-size parity checkers) give
    exactly the rows of the full assembly: same per-entry summation order, so
    bit-identical, including Dirichlet rows, boundary rows and the backflow
    tangent."""
    prob, d = load(name)
    for bf in (False, True):
        orc = ob.Restated(prob, tau_mode=int(d["tau_mode"]), pseudo_dt=d["pseudo_dt_eff"], backflow_tangent=bf)
        s = d["state"]
        nn, N = orc.nn, orc.N
        rows = np.random.default_rng(3).permutation(nn)[: max(5, nn // 3)].astype(np.int32)
        rows = np.concatenate([rows[rows != nn - 1], [nn - 1]]).astype(np.int32)
        full_r = orc.residual(s).reshape(nn, 4, N)
        assert np.array_equal(orc.residual_rows(s, rows), full_r[rows])
        full_p = orc.tangent(s)
        rp = orc.row_ptr
        want = np.concatenate([full_p[rp[A] * 8 * N: rp[A + 1] * 8 * N] for A in rows])
        assert np.array_equal(orc.tangent_rows(s, rows), want)
        m = orc.mass()
        y = d["y"]
        full_mv = orc.matvec(full_p, m, y).reshape(nn, 4, N)
        assert np.array_equal(orc.matvec_rows(want, m, y, rows), full_mv[rows])
    with pytest.raises(ob.OracleError):
        orc.residual_rows(s, np.array([0, 0], np.int32))


def test_row_subsets_resistance():
    """Row subsets with a resistance outlet equal the full restated residual."""
    prob, d = load("tube_m3_qp")
    outlet = [k for k, _ in prob.neumann][0]
    orc = ob.Restated(prob, tau_mode=int(d["tau_mode"]), pseudo_dt=d["pseudo_dt_eff"],
                      resistance={outlet: 1.1e4})
    s = d["state"]
    rows = np.arange(0, orc.nn, 3, dtype=np.int32)
    assert np.array_equal(orc.residual_rows(s, rows), orc.residual(s).reshape(orc.nn, 4, orc.N)[rows])
    p = orc.tangent(s)
    m = orc.mass()
    rp, N = orc.row_ptr, orc.N
    seg = np.concatenate([p[rp[A] * 8 * N: rp[A + 1] * 8 * N] for A in rows])
    assert np.array_equal(orc.matvec_rows(seg, m, d["y"], rows),
                          orc.matvec(p, m, d["y"]).reshape(orc.nn, 4, N)[rows])
