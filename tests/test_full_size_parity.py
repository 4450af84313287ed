"""Full-size parity on BASELINE configs 2, 3 and 4.

The complete CPU assembly of these meshes takes minutes to hours, so the
oracle computes a SAMPLE of rows instead: hbo_residual_rows /
hbo_tangent_rows / hbo_tangent_matvec_rows (oracle/hbgls_oracle.c) return
exactly the rows of the full restated assembly (same per-entry summation
order; pinned bit-for-bit against the full functions in
tests/test_oracle_pin.py).  The GPU path runs on the WHOLE mesh through the C
ABI; its residual, its P block rows (hbgpu_get_pvals_rows) and its L-matvec
are compared on ~1,100 sampled nodes: random interior nodes, the last nodes
(whose P.vals offsets exceed 2^31 doubles at config 4, Nm = 24), the
highest-valence nodes, Dirichlet and Neumann boundary nodes.

States: Newton iterate 0 (rest + Dirichlet + p0), Newton
iterate 1 (one GPU Newton step with the reference defaults) and a random
state for configs 2 and 3; the random-modes state ~N(0,1)/k^2 for config 4 at
Nm = 24 (N = 47) and Nm = 1.

Bars (north_star): residual, Jacobian rows and SpMV within 1e-12 relative
(normwise over the sampled rows, as test_assembly.cpp:264)."""
import numpy as np
import pytest

from oracle import bindings as ob
from paper_2411_14315_b200 import cases, meshgen
from paper_2411_14315_b200.mesh import NEUMANN

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0))


def sample_rows(mesh, row_ptr, n_random=1000, seed=0):
    nn = mesh.num_nodes
    rng = np.random.default_rng(seed)
    valence = np.diff(row_ptr)
    picks = [rng.choice(nn, size=min(n_random, nn), replace=False),
             np.arange(max(0, nn - 48), nn),                       # largest P offsets
             np.argsort(valence, kind="stable")[-16:],              # widest block rows
             np.flatnonzero(mesh.dirichlet)[:: max(1, int(mesh.dirichlet.sum()) // 24)][:24]]
    neu = [np.unique(p.facets) for p in mesh.patches if p.kind == NEUMANN]
    if neu:
        allneu = np.unique(np.concatenate(neu))
        picks.append(allneu[:: max(1, len(allneu) // 24)][:24])
    return np.unique(np.concatenate(picks)).astype(np.int32)


def gpu_ctx(prob, pseudo_dt):
    from paper_2411_14315_b200.hbgpu import GpuContext

    ctx = GpuContext(prob.mesh)
    ctx.set_basis(prob.modes, prob.period)
    ctx.set_fluid(prob.rho, prob.mu)
    ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
    ctx.set_assembly_config(0, pseudo_dt)
    return ctx


def check_state(ctx, orc, state, rows, row_ptr, mass, label, y_seed):
    N = orc.N
    nn = orc.nn
    r_gpu = ctx.assemble_residual(state).reshape(nn, 4, N)[rows]
    r_orc = orc.residual_rows(state, rows)
    e_r = rel(r_gpu, r_orc)
    ctx.assemble_tangent(state, download=False)
    p_gpu = ctx.pvals_rows(rows, row_ptr)
    p_orc = orc.tangent_rows(state, rows)
    e_p = rel(p_gpu, p_orc)
    y = cases.random_state(nn, N, y_seed)
    mv_gpu = ctx.matvec(y).reshape(nn, 4, N)[rows]
    mv_orc = orc.matvec_rows(p_orc, mass, y, rows)
    e_m = rel(mv_gpu, mv_orc)
    print(f"{label}: residual {e_r:.2e} tangent {e_p:.2e} matvec {e_m:.2e} ({len(rows)} rows)")
    assert e_r < TOL, (label, "residual", e_r)
    assert e_p < TOL, (label, "tangent", e_p)
    assert e_m < TOL, (label, "matvec", e_m)


def newton_iterate_1(prob, pseudo_dt):
    """One GPU Newton step from iterate 0 with the reference defaults
    (GMRES restart 200 / max 1000 / tol 0.03, hb_solver.cpp:150-213)."""
    from paper_2411_14315_b200.hbgpu import SolverConfig

    ctx = gpu_ctx(prob, pseudo_dt)
    sol = ctx.solve_harmonic(SolverConfig(pseudo_dt=pseudo_dt, max_newton_iters=1))
    assert len(sol.log.iters) >= 1
    return sol.state


@pytest.fixture(scope="module")
def cfg_meshes():
    return {}


def _mesh(cache, cfg):
    if cfg not in cache:
        cache[cfg] = meshgen.config_mesh(cfg)
    return cache[cfg]


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_size_configs_2_3(gpu, cfg_meshes, cfg):
    """Config 2 (944k-tet T-junction, N = 19) and config 3 (2.0M-tet curved
    stenosis, N = 31) at full size: iterate 0, iterate 1, random state."""
    prob = cases.config_problem(cfg, mesh=_mesh(cfg_meshes, cfg))
    from paper_2411_14315_b200.hbgpu import GpuContext  # noqa: F401

    ctx = gpu_ctx(prob, 0.05)
    dt = 0.05
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=dt)
    row_ptr = orc.row_ptr
    rp_gpu, _ = ctx.pattern()
    assert np.array_equal(rp_gpu, row_ptr)
    rows = sample_rows(prob.mesh, row_ptr, seed=cfg)
    mass = orc.mass()
    s0 = cases.initial_state(prob)
    check_state(ctx, orc, s0, rows, row_ptr, mass, f"cfg{cfg} iterate 0", 10 + cfg)
    s1 = newton_iterate_1(prob, dt)
    assert rel(s1, s0) > 1e-6  # the Newton step moved the state
    check_state(ctx, orc, s1, rows, row_ptr, mass, f"cfg{cfg} iterate 1", 20 + cfg)
    sr = cases.random_state(prob.mesh.num_nodes, prob.N, 100 + cfg, 2.0)
    check_state(ctx, orc, sr, rows, row_ptr, mass, f"cfg{cfg} random", 30 + cfg)


def test_full_size_config3_resistance(gpu, cfg_meshes):
    """Config 3 with the BASELINE resistance outlet (R = 1e4, SURVEY §8(f) row
    4, new physics restated in oracle/hbgls_oracle.c) at full size."""
    prob = cases.config_problem(3, mesh=_mesh(cfg_meshes, 3))
    outlets = {k: 1e4 for k, _ in prob.neumann}
    ctx = gpu_ctx(prob, 0.05)
    ctx.set_resistance(outlets)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.05, resistance=outlets)
    rows = sample_rows(prob.mesh, orc.row_ptr, n_random=400, seed=7)
    sr = cases.random_state(prob.mesh.num_nodes, prob.N, 203, 1.0)
    check_state(ctx, orc, sr, rows, orc.row_ptr, orc.mass(), "cfg3 resistance random", 41)


@pytest.mark.parametrize("modes", [24, 1])
def test_full_size_config4(gpu, cfg_meshes, modes):
    """Config 4 (700k-point Delaunay cube, 4.72M tets) at Nm = 24 (N = 47,
    P.vals = 34.6 GB, block offsets beyond 2^31 doubles) and Nm = 1."""
    mesh = _mesh(cfg_meshes, 4)
    N = 2 * modes - 1
    neu = [(k, np.full(N, 50.0)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    prob = cases.Problem(mesh, modes, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 3 * N), neu, 0.2)
    ctx = gpu_ctx(prob, 0.05)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.05)
    row_ptr = orc.row_ptr
    rows = sample_rows(mesh, row_ptr, seed=4)
    if modes == 24:
        # the sampled tail really exercises the 64-bit P offsets
        assert int(row_ptr[rows.max()]) * 8 * N > 2**31
    s = cases.random_modes_state(mesh.num_nodes, modes, 4)
    check_state(ctx, orc, s, rows, row_ptr, orc.mass(), f"cfg4 Nm={modes}", 50 + modes)
