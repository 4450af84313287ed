"""GPU time-stepping solver (hbgpu_solve_time) against the compiled reference's
solve_time (time_solver.cpp:269-485) on identical inputs, and the reference's
own time-solver properties (tests/test_time_solver.cpp).

Parity bar: with tight Newton (10 orders) and GMRES (1e-10) tolerances on both
sides, every snapshot of the last cycle agrees to 1e-8 relative L2 (velocity
and pressure) — the solves converge to the same discrete generalized-alpha
trajectory; only solver tolerances separate them."""
import os

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2411_14315_b200 import cases
from paper_2411_14315_b200.mesh import NEUMANN

pytestmark = pytest.mark.gpu
HAVE_REF = os.path.exists(ob.REF_SO)
PERIOD = 0.5


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def tube(h=0.15):
    if HAVE_REF:
        rm = ob.RefMesh.tube(0.3, 0.6, h)
        return rm, rm.to_mesh()
    from paper_2411_14315_b200 import meshgen

    return None, meshgen.hex_cylinder(0.3, 0.6, 3, 3, 4)


def gpu_time_ctx(mesh, h_out):
    from paper_2411_14315_b200.hbgpu import GpuContext

    ctx = GpuContext(mesh)
    ctx.set_basis(1, PERIOD)
    ctx.set_fluid(1.06, 0.04)
    ctx.set_bcs(None, [(k, np.array([h_out])) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN], 0.2)
    return ctx


def time_cfg(steps, cycles, orders=10.0, max_newton=12, tol=1e-10, steady=False):
    from paper_2411_14315_b200.hbgpu import KrylovConfig, TimeSolverConfig

    return TimeSolverConfig(steps_per_cycle=steps, cycles=cycles, newton_tol_orders=orders,
                            max_newton_iters=max_newton, krylov=KrylovConfig(200, 1000, tol), steady=steady)


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference (oracle/_ref) missing")
@pytest.mark.parametrize("h_out", [-20.0, 0.0])
def test_time_solve_matches_reference(gpu, h_out):
    rm, mesh = tube()
    fn = cases.time_dirichlet(mesh, mesh.patch_index("inlet"), 2.0, [0.2, -0.1], [0.1, 0.05], PERIOD)
    ref = ob.RefCtx(rm, 1, PERIOD)
    ref.set_bcs(None, [(k, np.array([h_out])) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN], 0.2)
    r = ref.solve_time(fn, PERIOD, steps=20, cycles=2, orders=10.0, max_newton=12, tol=1e-10)
    g = gpu_time_ctx(mesh, h_out).solve_time(fn, time_cfg(20, 2))
    assert g.total_steps == r["total_steps"] == 40
    assert g.u.shape == r["u"].shape and g.p.shape == r["p"].shape
    for j in range(g.u.shape[0]):
        assert rel(g.u[j], r["u"][j]) < 1e-8, j
        assert rel(g.p[j], r["p"][j]) < 1e-8, j
    assert abs(g.cycle_change - r["cycle_change"]) <= 1e-6 * abs(r["cycle_change"])
    assert abs(g.omega_hat_last - r["omega_hat_last"]) <= 1e-6 * abs(r["omega_hat_last"])
    assert abs(g.total_newton_iters - r["total_newton_iters"]) <= 0.05 * r["total_newton_iters"]


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference (oracle/_ref) missing")
def test_time_solve_reference_defaults(gpu):
    """Default tolerances (3 orders, 8 Newton, GMRES 0.03): the same Newton and
    GMRES decisions on both sides, so the same trajectory to round-off (measured
    ~1e-14 on this tube)."""
    rm, mesh = tube()
    fn = cases.time_dirichlet(mesh, mesh.patch_index("inlet"), 2.0, [0.2, -0.1], [0.1, 0.05], PERIOD)
    ref = ob.RefCtx(rm, 1, PERIOD)
    ref.set_bcs(None, [(k, np.array([-20.0])) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN], 0.2)
    r = ref.solve_time(fn, PERIOD, steps=25, cycles=2)
    g = gpu_time_ctx(mesh, -20.0).solve_time(fn, time_cfg(25, 2, orders=3.0, max_newton=8, tol=0.03))
    for j in range(g.u.shape[0]):
        assert rel(g.u[j], r["u"][j]) < 1e-10, j
        assert rel(g.p[j], r["p"][j]) < 1e-10, j
    assert g.total_newton_iters == r["total_newton_iters"]


def test_time_zero_forcing_stays_zero(gpu):
    """test_time_solver.cpp:45-60: no inflow, zero traction -> identically zero."""
    _, mesh = tube()
    nn = mesh.num_nodes
    z = np.zeros(nn * 3)
    sol = gpu_time_ctx(mesh, 0.0).solve_time(lambda t: (z, z), time_cfg(50, 1, orders=3.0, max_newton=8,
                                                                           tol=0.03))
    assert sol.total_steps == 50
    assert np.all(sol.u == 0.0) and np.all(sol.p == 0.0)


def test_time_steady_equals_harmonic_n1(gpu):
    """Shared-discretization anchor (test_time_solver.cpp:62-83): steady mode of
    the time solver equals the N = 1 harmonic-balance solve, both on the GPU."""
    from paper_2411_14315_b200.hbgpu import KrylovConfig, SolverConfig

    _, mesh = tube(0.12)
    inlet = mesh.patch_index("inlet")
    fn = cases.time_dirichlet(mesh, inlet, 1.5, [], [], PERIOD)
    ctx = gpu_time_ctx(mesh, 0.0)
    g0, _ = fn(0.0)
    nn = mesh.num_nodes
    ctx.set_bcs(g0.reshape(nn * 3), [(k, np.array([0.0])) for k, p in enumerate(mesh.patches)
                                      if p.kind == NEUMANN], 0.2)
    hb = ctx.solve_harmonic(SolverConfig(newton_tol_orders=7.0, max_newton_iters=200,
                                         krylov=KrylovConfig(200, 1000, 1e-6)))
    assert hb.log.converged
    ts = ctx.solve_time(fn, time_cfg(1, 1, orders=7.0, max_newton=200, tol=1e-6, steady=True))
    s = hb.state.reshape(nn, 4)
    assert rel(ts.u[0], s[:, :3].reshape(-1)) < 1e-5
    assert rel(ts.p[0], s[:, 3]) < 1e-4


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference (oracle/_ref) missing")
def test_time_steady_matches_reference(gpu):
    rm, mesh = tube()
    fn = cases.time_dirichlet(mesh, mesh.patch_index("inlet"), 1.5, [], [], PERIOD)
    ref = ob.RefCtx(rm, 1, PERIOD)
    ref.set_bcs(None, [(k, np.array([-10.0])) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN], 0.2)
    r = ref.solve_time(fn, PERIOD, steps=1, cycles=1, orders=10.0, max_newton=40, tol=1e-10, steady=True)
    g = gpu_time_ctx(mesh, -10.0).solve_time(fn, time_cfg(1, 1, orders=10.0, max_newton=40, tol=1e-10,
                                                          steady=True))
    assert rel(g.u[0], r["u"][0]) < 1e-8
    assert rel(g.p[0], r["p"][0]) < 1e-8


def test_time_needs_n1_basis(gpu):
    from paper_2411_14315_b200.hbgpu import GpuContext

    _, mesh = tube()
    ctx = GpuContext(mesh)
    ctx.set_basis(3, PERIOD)
    z = np.zeros(mesh.num_nodes * 3)
    with pytest.raises(ValueError):
        ctx.solve_time(lambda t: (z, z), time_cfg(5, 1))


def _time_problem(mesh, h_out):
    return cases.Problem(mesh, 1, PERIOD, 1.06, 0.04, np.zeros(mesh.num_nodes * 3),
                         [(k, np.array([h_out])) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN], 0.2)


@pytest.mark.parametrize("which", ["tube", "config0"])
def test_time_operators_match_restatement(gpu, which):
    """time_residual / time_tangent kernels vs the plain-C restatement of
    time_solver.cpp:58-254 at 1e-12, on a random state (both omega_hat regimes,
    generalized-alpha and steady factors)."""
    if which == "tube":
        _, mesh = tube()
    else:
        mesh = cases.config_problem(0).mesh
    prob = _time_problem(mesh, -20.0)
    orc = ob.Restated(prob)
    ctx = gpu_time_ctx(mesh, -20.0)
    rng = np.random.default_rng(7)
    nn = mesh.num_nodes
    u, ud, p = rng.uniform(-2, 2, nn * 3), rng.uniform(-20, 20, nn * 3), rng.uniform(-50, 50, nn)
    for om in (0.0, 3.7):
        assert rel(ctx.time_residual(u, ud, p, om), orc.time_residual(u, ud, p, om)) < 1e-12
        for am, fg in ((0.9166666, 0.00138), (0.0, 1.0)):
            assert rel(ctx.time_tangent(u, om, am, fg), orc.time_tangent(u, om, am, fg)) < 1e-12
