"""GPU parity: the CUDA hot path (through the C ABI) against the oracles.

Bars (BASELINE.json north_star): residual / Jacobian / SpMV <= 1e-12 relative
(fp64, normwise as test_assembly.cpp:264); pattern and DOF indexing
bit-exact.  The oracles are the plain-C restatement (always) and the compiled
reference (oracle/_ref/libhbref.so, when present)."""
import os

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2411_14315_b200 import cases
from paper_2411_14315_b200.cases import Problem
from paper_2411_14315_b200.mesh import NEUMANN

pytestmark = pytest.mark.gpu
TOL = 1e-12
HAVE_REF = os.path.exists(ob.REF_SO)


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def gpu_ctx(prob, tau_mode=0, pseudo_dt=float("inf")):
    from paper_2411_14315_b200.hbgpu import GpuContext

    ctx = GpuContext(prob.mesh)
    ctx.set_basis(prob.modes, prob.period)
    ctx.set_fluid(prob.rho, prob.mu)
    ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
    ctx.set_assembly_config(tau_mode, pseudo_dt)
    return ctx


def tube_problem(modes, radius=0.5, length=1.0, h=0.34, seed=1, period=0.8, traction=True):
    rm = ob.RefMesh.tube(radius, length, h) if HAVE_REF else None
    if rm is not None:
        mesh = rm.to_mesh()
    else:
        from paper_2411_14315_b200 import meshgen

        mesh = meshgen.hex_cylinder(radius, length, 3, 3, 4)
    N = 2 * modes - 1
    rng = np.random.default_rng(seed)
    neu = [(k, (rng.uniform(-1, 1, N) * 100 + 5) if traction else np.zeros(N))
           for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    g = rng.uniform(-1, 1, mesh.num_nodes * 3 * N)
    return Problem(mesh, modes, period, 1.06, 0.04, g, neu, 0.2)


CASES = [(m, tau, pdt) for m in (1, 3, 4) for tau in (0, 1) for pdt in (0.3, float("inf"))]


@pytest.mark.parametrize("modes,tau,pdt", CASES)
def test_small_tube_all_ops(gpu, modes, tau, pdt):
    prob = tube_problem(modes)
    ctx = gpu_ctx(prob, tau, pdt)
    orc = ob.Restated(prob, tau_mode=tau, pseudo_dt=pdt)
    nn, N = prob.mesh.num_nodes, prob.N
    s = cases.random_state(nn, N, 11)
    r_gpu = ctx.assemble_residual(s)
    r_orc = orc.residual(s)
    assert rel(r_gpu, r_orc) < TOL
    p_gpu = ctx.assemble_tangent(s)
    p_orc = orc.tangent(s)
    assert rel(p_gpu, p_orc) < TOL
    m_gpu = ctx.assemble_mass()
    m_orc = orc.mass()
    assert np.array_equal(m_gpu, m_orc) or rel(m_gpu, m_orc) < 1e-15
    y = cases.random_state(nn, N, 12)
    assert rel(ctx.matvec(y), orc.matvec(p_orc, m_orc, y)) < TOL
    assert rel(ctx.bsr_matvec(y), orc.bsr_matvec(p_orc, y)) < TOL
    inv_gpu, deg_gpu = ctx.jacobi()
    inv_orc, deg_orc = orc.jacobi(p_gpu)
    assert deg_gpu == deg_orc
    assert rel(inv_gpu, inv_orc) < TOL
    if HAVE_REF:
        ref = ob.ref_context(prob, tau, pdt)
        assert rel(r_gpu, ref.residual(s)) < TOL
        assert rel(p_gpu, ref.tangent(s)) < TOL
        assert rel(ctx.matvec(y), ref.matvec(y)) < TOL


@pytest.mark.parametrize("name", ["tube_m3_qp", "tube_m4_mean", "tube_m1_steady", "bifurcation_m3"])
def test_against_golden_fixtures(gpu, name):
    """GPU path vs the committed outputs of the compiled reference."""
    from goldens import load
    from paper_2411_14315_b200.hbgpu import GpuContext, KrylovConfig

    prob, d = load(name)
    # geometry passed as the reference's ElementGeometry array (zero-copy drop-in)
    ctx = GpuContext(prob.mesh, geometry=d["geometry"])
    ctx.set_basis(prob.modes, prob.period)
    ctx.set_fluid(prob.rho, prob.mu)
    ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
    ctx.set_assembly_config(int(d["tau_mode"]), d["pseudo_dt_eff"])
    rp, ci = ctx.pattern()
    assert np.array_equal(rp, d["row_ptr"]) and np.array_equal(ci, d["col_idx"])
    assert rel(ctx.assemble_residual(d["state"]), d["residual"]) < TOL
    assert rel(ctx.assemble_tangent(d["state"]), d["pvals"]) < TOL
    assert rel(ctx.assemble_mass(), d["mass"]) < 1e-15
    assert rel(ctx.matvec(d["y"]), d["matvec"]) < TOL
    ctx.set_pvals(d["pvals"])
    inv, deg = ctx.jacobi()
    assert deg == int(d["degenerate"]) and rel(inv, d["inv_diag"]) < 1e-15
    res = ctx.gmres(d["matvec"], KrylovConfig(restart=40, max_iters=400, tolerance=1e-9))
    assert res.relative_residual <= 1e-9 or res.status == 1
    assert abs(res.iterations - int(d["gmres_iters"])) <= max(3, 0.05 * int(d["gmres_iters"]))
    if float(d["gmres_relres"]) <= 1e-9:  # both converged: solutions agree to ~kappa * tol
        assert rel(res.x, d["gmres_x"]) < 1e-6


@pytest.mark.parametrize("modes", [1, 3])
def test_backflow_in_tangent(gpu, modes):
    """AssemblyConfig::backflow_in_tangent (assembly.cpp:612-657)."""
    prob = tube_problem(modes, h=0.25)
    ctx = gpu_ctx(prob, 0, 0.3)
    ctx.set_assembly_config(0, 0.3, 1.5, True)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.3, backflow_tangent=True)
    s = cases.random_state(prob.mesh.num_nodes, prob.N, 31)
    p_gpu = ctx.assemble_tangent(s)
    p_orc = orc.tangent(s)
    assert rel(p_gpu, p_orc) < TOL
    assert rel(p_orc, ob.Restated(prob, tau_mode=0, pseudo_dt=0.3).tangent(s)) > 1e-8  # term is active
    if HAVE_REF:
        ref = ob.ref_context(prob, 0, 0.3)
        ref.set_cfg(0, 0.3, 1.5, True)
        assert rel(p_gpu, ref.tangent(s)) < TOL


@pytest.mark.parametrize("modes", [1, 4, 24])
def test_delaunay_cube_operator(gpu, modes):
    """Config-4 style mesh (Delaunay, high-valence hull nodes, Morton order)
    at N up to 47: exercises the time-sample tiling of the tangent kernel."""
    from paper_2411_14315_b200 import meshgen

    mesh = meshgen.cube_delaunay(4000, seed=11)
    N = 2 * modes - 1
    neu = [(k, np.full(N, 50.0)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    prob = Problem(mesh, modes, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 3 * N), neu, 0.2)
    ctx = gpu_ctx(prob, 0, 0.05)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.05)
    s = cases.random_modes_state(mesh.num_nodes, modes, 3)
    assert rel(ctx.assemble_residual(s), orc.residual(s)) < TOL
    p_gpu = ctx.assemble_tangent(s)
    p_orc = orc.tangent(s)
    assert rel(p_gpu, p_orc) < TOL
    y = cases.random_state(mesh.num_nodes, N, 5)
    assert rel(ctx.matvec(y), orc.matvec(p_orc, orc.mass(), y)) < TOL
    rp, ci = ctx.pattern()
    assert np.array_equal(ci, orc.col_idx)


@pytest.mark.parametrize("tile", ["1", "2", "4"])
@pytest.mark.parametrize("modes", [2, 4, 10])
def test_residual_tile_widths(gpu, monkeypatch, tile, modes):
    """Every residual tile width (samples per tile; HBGPU_RES_TILE, read when
    the basis is set) against the oracle, including partial last tiles
    (N = 3, 7, 19) and the sample-pair gathers of the even widths."""
    from paper_2411_14315_b200 import meshgen

    monkeypatch.setenv("HBGPU_RES_TILE", tile)
    mesh = meshgen.cube_delaunay(3000, seed=9)
    N = 2 * modes - 1
    neu = [(k, np.full(N, 50.0)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    prob = Problem(mesh, modes, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 3 * N), neu, 0.2)
    ctx = gpu_ctx(prob, 0, 0.05)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.05)
    s = cases.random_modes_state(mesh.num_nodes, modes, 13)
    assert rel(ctx.assemble_residual(s), orc.residual(s)) < TOL


@pytest.mark.parametrize("width", ["64", "256"])
def test_tangent_pipe_widths(gpu, monkeypatch, width):
    """The persistent tangent pipeline at forced CTA widths (HBGPU_TAN_WIDTH)."""
    monkeypatch.setenv("HBGPU_TAN_WIDTH", width)
    prob = tube_problem(4)
    ctx = gpu_ctx(prob, 0, 0.3)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.3)
    s = cases.random_modes_state(prob.mesh.num_nodes, 4, 17)
    assert rel(ctx.assemble_tangent(s), orc.tangent(s)) < TOL


@pytest.mark.parametrize("mesh_kind,modes,tau", [("tube", 3, 0), ("tube", 4, 1), ("delaunay", 4, 0),
                                                  ("delaunay", 24, 0)])
def test_tangent_row_kernel_fallback(gpu, monkeypatch, mesh_kind, modes, tau):
    """The tiled row kernel (used for rows whose neighbour records do not fit
    the persistent pipeline's shared memory) against the oracle; forced with
    the HBGPU_TANGENT_KERNEL=rows test knob, read when the basis is set."""
    from paper_2411_14315_b200 import meshgen

    monkeypatch.setenv("HBGPU_TANGENT_KERNEL", "rows")
    if mesh_kind == "tube":
        prob = tube_problem(modes)
    else:
        mesh = meshgen.cube_delaunay(3000, seed=5)
        N = 2 * modes - 1
        neu = [(k, np.full(N, 50.0)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
        prob = Problem(mesh, modes, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 3 * N), neu, 0.2)
    ctx = gpu_ctx(prob, tau, 0.3)
    orc = ob.Restated(prob, tau_mode=tau, pseudo_dt=0.3)
    s = cases.random_modes_state(prob.mesh.num_nodes, modes, 7)
    assert rel(ctx.assemble_tangent(s), orc.tangent(s)) < TOL


def test_combined_assemble_host_call(gpu):
    """hbgpu_assemble (one upload, residual to the host, P kept on the device)
    equals the separate calls: residual vs the oracle, and the L-matvec that
    follows uses the freshly assembled P."""
    prob = tube_problem(4)
    ctx = gpu_ctx(prob, 0, 0.3)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.3)
    nn, N = prob.mesh.num_nodes, prob.N
    s = cases.random_state(nn, N, 21)
    r = ctx.assemble(s)
    assert rel(r, orc.residual(s)) < TOL
    ctx.assemble_mass()
    y = cases.random_state(nn, N, 22)
    assert rel(ctx.matvec(y), orc.matvec(orc.tangent(s), orc.mass(), y)) < TOL


def test_pattern_bit_exact(gpu):
    from paper_2411_14315_b200 import meshgen

    mesh = meshgen.hex_cylinder(0.3, 2.0, 6, 6, 20)
    prob = Problem(mesh, 2, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 9), [], 0.2)
    ctx = gpu_ctx(prob)
    rp, ci = ctx.pattern()
    rp2, ci2 = ob.restated_pattern(mesh.num_nodes, mesh.conn)
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2)
    if HAVE_REF:
        rp3, ci3 = ob.RefMesh.from_mesh(mesh).pattern()
        assert np.array_equal(rp, rp3) and np.array_equal(ci, ci3)
    g = ctx.geometry()
    assert np.abs(g - ob.restated_geometry(mesh.xyz, mesh.conn)).max() <= 1e-12 * np.abs(g).max()


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_config_residual_tangent_matvec(gpu, cfg):
    """Configs 0/1 at full size; configs 2/3 (T-junction Delaunay, curved
    stenosis) on reduced meshes of the same generators, full N (19 / 31)."""
    from paper_2411_14315_b200 import meshgen

    small = {2: lambda: meshgen.tjunction_delaunay(20000, seed=2), 3: lambda: meshgen.stenosis_tube(10, 120)}
    prob = cases.config_problem(cfg, mesh=small[cfg]() if cfg in small else None)
    nn, N = prob.mesh.num_nodes, prob.N
    ctx = gpu_ctx(prob, 0, 0.05)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.05)
    for s in (cases.initial_state(prob), cases.random_state(nn, N, 100 + cfg, 2.0)):
        assert rel(ctx.assemble_residual(s), orc.residual(s)) < TOL
        p_gpu = ctx.assemble_tangent(s)
        p_orc = orc.tangent(s)
        assert rel(p_gpu, p_orc) < TOL
    y = cases.random_state(nn, N, 7)
    assert rel(ctx.matvec(y), orc.matvec(p_orc, orc.mass(), y)) < TOL


def test_gmres_scaled_residual(gpu):
    """GMRES: the CPU operator's scaled residual ||S(b - L x_gpu)|| / ||S b||
    meets the tolerance; same iteration-count
    ballpark as the reference."""
    from paper_2411_14315_b200.hbgpu import KrylovConfig

    prob = tube_problem(3, h=0.25, traction=False)
    ctx = gpu_ctx(prob, 0, 0.3)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.3)
    s = cases.random_state(prob.mesh.num_nodes, prob.N, 21, 0.5)
    p = ctx.assemble_tangent(s)
    m = orc.mass()
    inv, _ = ctx.jacobi()
    b = cases.random_state(prob.mesh.num_nodes, prob.N, 22)
    for tol in (1e-3, 1e-8):
        res = ctx.gmres(b, KrylovConfig(restart=60, max_iters=2000, tolerance=tol))
        assert res.status == 0
        scale = np.sqrt(np.abs(inv))
        rr = np.linalg.norm(scale * (b - orc.matvec(p, m, res.x))) / np.linalg.norm(scale * b)
        assert rr <= tol * 1.0001
        assert np.all(np.diff(res.history) <= 1e-14)
        ref = orc.gmres(p, m, b, inv, restart=60, max_iters=2000, tol=tol)
        assert abs(ref["iterations"] - res.iterations) <= max(3, 0.1 * ref["iterations"])


def test_gmres_identity_zero_and_stagnation(gpu):
    from paper_2411_14315_b200.hbgpu import KrylovConfig

    prob = tube_problem(2, traction=False)
    ctx = gpu_ctx(prob)
    n = ctx.state_len
    nnz = ctx.nnz
    N = prob.N
    # identity operator: P = I block diagonal, no C (mass zero is not settable;
    # use N = 3 with velocity identity and pressure identity on the diagonal)
    rp, ci = ctx.pattern()
    vals = np.zeros((nnz, 8, N))
    diag = np.array([np.searchsorted(ci[rp[a]:rp[a + 1]], a) + rp[a] for a in range(len(rp) - 1)])
    vals[diag, 0, :] = 1.0
    vals[diag, 7, :] = 1.0
    ctx.set_pvals(vals.reshape(-1))
    b = cases.random_state(prob.mesh.num_nodes, N, 5)
    # zero rhs
    res0 = ctx.gmres(np.zeros(n), KrylovConfig())
    assert res0.iterations == 0 and res0.relative_residual == 0.0 and not res0.x.any()
    # a P-only operator on Dirichlet-free rows is I + H(x)mass; checked against the restatement
    orc = ob.Restated(prob)
    m = orc.mass()
    res = ctx.gmres(b, KrylovConfig(tolerance=1e-10, restart=80, max_iters=800))
    assert res.status == 0
    assert rel(orc.matvec(vals.reshape(-1), m, res.x), b) < 1e-9


def _modes(state, nn, N, comps):
    """PeriodicSignal::coefficients (spectral.cpp:35-50): c_m = (1/N) sum_n v_n e^{-2 pi i m n/N}."""
    v = state.reshape(nn, 4, N)[:, comps, :]
    return np.fft.fft(v, axis=-1) / N


@pytest.mark.skipif(not HAVE_REF, reason="compiled reference absent")
def test_converged_solve_matches_reference(gpu):
    """Converged periodic velocity / pressure within 1e-8 relative L2, in time
    samples and in Fourier modes, with tight tolerances on both sides
    (Newton 10 orders, GMRES 1e-10, CFL 3)."""
    from paper_2411_14315_b200.hbgpu import GpuContext, KrylovConfig, SolverConfig

    rm = ob.RefMesh.tube(0.3, 1.5, 0.15)
    mesh = rm.to_mesh()
    M, N = 3, 5
    q = cases.flow_samples(2.0, [0.2, -0.1], [0.1, 0.05], M, 1.0)
    g = cases.parabolic_dirichlet(mesh, mesh.patch_index("inlet"), q)
    neu = [(k, np.full(N, -100.0)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    prob = Problem(mesh, M, 1.0, 1.06, 0.04, g, neu, 0.2)
    rc = ob.ref_context(prob)
    dt = 3.0 * rc.suggest_pseudo_dt()
    ref = rc.solve(pseudo_dt=dt, orders=10, max_newton=300, restart=200, max_iters=5000, tol=1e-10)
    assert ref["converged"]
    ctx = GpuContext(mesh)
    ctx.set_basis(M, 1.0)
    ctx.set_fluid(1.06, 0.04)
    ctx.set_bcs(g, neu, 0.2)
    sol = ctx.solve_harmonic(SolverConfig(pseudo_dt=dt, newton_tol_orders=10, max_newton_iters=300,
                                          krylov=KrylovConfig(200, 5000, 1e-10)))
    assert sol.log.converged
    assert abs(sol.cfl - ref["cfl"]) < 1e-12 * ref["cfl"]
    nn = mesh.num_nodes
    su, sr = sol.state.reshape(nn, 4, N), ref["state"].reshape(nn, 4, N)
    assert rel(su[:, :3], sr[:, :3]) < 1e-8
    assert rel(su[:, 3], sr[:, 3]) < 1e-8
    assert rel(_modes(sol.state, nn, N, slice(0, 3)), _modes(ref["state"], nn, N, slice(0, 3))) < 1e-8
    assert rel(_modes(sol.state, nn, N, 3), _modes(ref["state"], nn, N, 3)) < 1e-8
    # same Newton trajectory length within a couple of iterations
    assert abs(len(sol.log.iters) - len(ref["res"])) <= 3


def test_cpp_adapter_against_reference(gpu):
    """The C++ drop-in adapter (integration/hbflow_gpu.cpp, reference
    signatures) on the reference's own build_case tube, side by side with the
    reference functions: residual, tangent, mass, matvec, Jacobi, GMRES and a
    tight converged solve."""
    import json
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "integration", "_build", "adapter_demo")
    if not os.path.exists(exe):
        pytest.skip("adapter demo not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert out.returncode == 0 and line["ok"], line


def test_solver_is_deterministic(gpu):
    """Bit-identical convergence history and state across runs (test_hb_solver.cpp:124-141)."""
    from paper_2411_14315_b200.hbgpu import GpuContext, SolverConfig

    prob = cases.config_problem(0)
    runs = []
    for _ in range(2):
        ctx = GpuContext(prob.mesh)
        ctx.set_basis(prob.modes, prob.period)
        ctx.set_fluid(prob.rho, prob.mu)
        ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
        runs.append(ctx.solve_harmonic(SolverConfig(max_newton_iters=5)))
    assert np.array_equal(runs[0].state, runs[1].state)
    assert np.array_equal(runs[0].log.res, runs[1].log.res)
    assert np.array_equal(runs[0].log.linear_iters, runs[1].log.linear_iters)


@pytest.mark.parametrize("modes", [1, 3])
def test_singular_tau_is_domain_error(gpu, modes):
    """compute_tau throws std::domain_error (assembly.cpp:51-53)."""
    prob = tube_problem(modes)
    from paper_2411_14315_b200.hbgpu import GpuContext

    ctx = GpuContext(prob.mesh)
    ctx.set_basis(modes, 1.0)
    ctx.set_fluid(1.0, 1e-300)  # nu^2 underflows to zero
    s = np.zeros(ctx.state_len)
    with pytest.raises(ArithmeticError):
        ctx.assemble_residual(s)


@pytest.mark.parametrize("lanes", ["0", "1", "4"])
@pytest.mark.parametrize("modes", [1, 3, 4])
def test_matvec_kernel_lanes(gpu, monkeypatch, modes, lanes):
    """Both L-matvec kernels for N > 1 — one thread per (row, sample), and four
    lanes per (row, sample) combined in fixed order (HBGPU_MV_LANES, read at
    context creation; 0 = automatic) — and the four-lane N = 1 kernel against
    the restatement: different block summation orders, same 1e-12 bar;
    bitwise repeatable."""
    monkeypatch.setenv("HBGPU_MV_LANES", lanes)
    prob = tube_problem(modes, h=0.25)
    ctx = gpu_ctx(prob, 0, 0.3)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.3)
    s = cases.random_state(prob.mesh.num_nodes, prob.N, 21)
    p = ctx.assemble_tangent(s)
    m = orc.mass()
    y = cases.random_state(prob.mesh.num_nodes, prob.N, 22)
    out = ctx.matvec(y)
    assert rel(out, orc.matvec(p, m, y)) < TOL
    assert rel(ctx.bsr_matvec(y), orc.bsr_matvec(p, y)) < TOL
    assert np.array_equal(out, ctx.matvec(y))


@pytest.mark.parametrize("modes", [1, 3])
def test_resistance_outlet(gpu, modes):
    """Resistance outlet (BASELINE config 3, new physics
    restated in oracle/hbgls_oracle.c): residual and TangentOperator::matvec
    with the R Q(u) traction vs the restatement at 1e-12; the BSR matvec (P
    only) is unchanged; the matvec's extra part is exactly R b b^T y."""
    prob = tube_problem(modes, h=0.25)
    outlet = [k for k, p in enumerate(prob.mesh.patches) if p.kind == NEUMANN][0]
    R = 1.3e4
    ctx = gpu_ctx(prob, 0, 0.3)
    ctx.set_resistance({outlet: R})
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.3, resistance={outlet: R})
    orc0 = ob.Restated(prob, tau_mode=0, pseudo_dt=0.3)
    nn, N = prob.mesh.num_nodes, prob.N
    s = cases.random_state(nn, N, 31)
    r = ctx.assemble_residual(s)
    assert rel(r, orc.residual(s)) < TOL
    assert rel(r, orc0.residual(s)) > 1e-6  # the term is really there
    p = ctx.assemble_tangent(s)
    m = orc.mass()
    y = cases.random_state(nn, N, 32)
    out = ctx.matvec(y)
    assert rel(out, orc.matvec(p, m, y)) < TOL
    assert rel(ctx.bsr_matvec(y), orc.bsr_matvec(p, y)) < TOL
    # the operator's outlet part is the derivative of the residual's (linear in u,
    # Dirichlet columns masked)
    d_l = out - orc0.matvec(p, m, y)
    yf = y.copy().reshape(nn, 4, N)
    yf[prob.mesh.dirichlet.astype(bool)] = 0.0
    d_rf = (orc.residual(s + yf.reshape(-1)) - orc0.residual(s + yf.reshape(-1))) - (orc.residual(s) - orc0.residual(s))
    assert rel(d_l, d_rf) < 1e-10
    ctx.set_resistance({outlet: 0.0})
    assert rel(ctx.assemble_residual(s), orc0.residual(s)) < TOL


def test_resistance_outlet_solve(gpu):
    """A harmonic solve with a resistance outlet converges (GPU Newton + GMRES
    on the operator with the rank-one outlet coupling) to a root of the
    restated residual with the same outlet."""
    from paper_2411_14315_b200.hbgpu import KrylovConfig, SolverConfig

    prob = tube_problem(3, h=0.25, traction=False)
    outlet = [k for k, p in enumerate(prob.mesh.patches) if p.kind == NEUMANN][0]
    g = cases.parabolic_dirichlet(prob.mesh, prob.mesh.patch_index("inlet"),
                                  cases.flow_samples(2.0, [0.2, -0.1], [0.1, 0.05], 3, prob.period))
    prob = cases.Problem(prob.mesh, 3, prob.period, 1.06, 0.04, g, prob.neumann, 0.2)
    ctx = gpu_ctx(prob)
    ctx.set_resistance({outlet: 1e4})
    sol = ctx.solve_harmonic(SolverConfig(newton_tol_orders=8.0, max_newton_iters=200,
                                          krylov=KrylovConfig(200, 2000, 1e-9)))
    assert sol.log.converged
    orc = ob.Restated(prob, resistance={outlet: 1e4}, pseudo_dt=0.0)
    r = orc.residual(sol.state)
    r0 = orc.residual(cases.initial_state(prob))
    assert np.linalg.norm(r) <= 1e-7 * np.linalg.norm(r0)
    # outlet pressure follows R Q: the mean outlet pressure is ~R times the mean inflow (2 mL/s)
    pr = sol.state.reshape(prob.mesh.num_nodes, 4, prob.N)[:, 3, :]
    onodes = np.unique(prob.mesh.patches[outlet].facets)
    assert 0.5 * 2e4 < pr[onodes].mean() < 1.5 * 2e4


def test_error_paths(gpu):
    """The reference's exceptions through the C ABI: degenerate element ->
    GeometryError (mesh.cpp:173-174, the device geometry pass), bad basis / fluid
    -> ParseError (spectral.cpp:19-22, assembly.cpp:38-41), Neumann data on a
    missing patch -> invalid_argument (the reference would index out of range).
    Neumann data on a Dirichlet patch is accepted, as in the reference
    (accumulate_boundary_terms does not check the kind): it only touches
    constrained rows, which are zeroed."""
    from paper_2411_14315_b200 import meshgen
    from paper_2411_14315_b200.hbgpu import GpuContext
    from paper_2411_14315_b200.mesh import GeometryError, ParseError

    mesh = meshgen.hex_cylinder(0.3, 1.0, 2, 2, 3)
    mesh.finalize()
    bad = mesh.xyz.copy()
    e0 = mesh.conn[0]
    bad[e0[3]] = bad[e0[0]] + 0.5 * (bad[e0[1]] - bad[e0[0]])  # collapse element 0
    mesh.xyz = bad
    with pytest.raises(GeometryError):
        GpuContext(mesh)
    mesh = meshgen.hex_cylinder(0.3, 1.0, 2, 2, 3)
    ctx = GpuContext(mesh)
    with pytest.raises(ParseError):
        ctx.set_basis(0, 1.0)
    ctx.set_basis(2, 1.0)
    with pytest.raises(ParseError):
        ctx.set_fluid(-1.0, 0.04)
    ctx.set_bcs(None, [(mesh.patch_index("wall"), np.ones(3))], 0.2)
    with pytest.raises(ValueError):
        ctx.set_bcs(None, [(len(mesh.patches) + 3, np.zeros(3))], 0.2)


def test_all_dirichlet_boundary(gpu):
    """No Neumann patch at all (every boundary node constrained): residual,
    tangent and L-matvec parity; Dirichlet velocity rows zero, pressure rows kept."""
    from paper_2411_14315_b200 import meshgen
    from paper_2411_14315_b200.mesh import DIRICHLET, Mesh, Patch

    m0 = meshgen.hex_cylinder(0.4, 1.0, 3, 3, 4)
    mesh = Mesh(xyz=m0.xyz, conn=m0.conn,
                patches=[Patch(p.name, DIRICHLET, p.facets) for p in m0.patches])
    mesh.finalize()
    N = 5
    g = np.random.default_rng(3).uniform(-1, 1, mesh.num_nodes * 3 * N)
    prob = cases.Problem(mesh, 3, 1.0, 1.06, 0.04, g, [], 0.2)
    ctx = gpu_ctx(prob, 0, 0.2)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.2)
    s = cases.random_state(mesh.num_nodes, N, 51)
    r = ctx.assemble_residual(s)
    assert rel(r, orc.residual(s)) < TOL
    rv = r.reshape(mesh.num_nodes, 4, N)
    assert np.all(rv[mesh.dirichlet.astype(bool), :3] == 0.0)
    p = ctx.assemble_tangent(s)
    assert rel(p, orc.tangent(s)) < TOL
    y = cases.random_state(mesh.num_nodes, N, 52)
    assert rel(ctx.matvec(y), orc.matvec(p, orc.mass(), y)) < TOL


@pytest.mark.parametrize("restart", [8, 600, 1000])
def test_gmres_device_and_host_loops(gpu, monkeypatch, restart):
    """The device-resident GMRES cycle (batched steps, device Arnoldi kernel;
    restart 600 needs the large shared-memory opt-in) and the host-driven loop
    (restart 1000 exceeds the Arnoldi kernel's shared memory; HBGPU_GMRES_HOST
    forces it) reach the same solution, iteration counts and history."""
    from paper_2411_14315_b200.hbgpu import KrylovConfig

    prob = tube_problem(3, h=0.25, traction=False)
    ctx = gpu_ctx(prob, 0, 0.3)
    s = cases.random_state(prob.mesh.num_nodes, prob.N, 61, 0.5)
    ctx.assemble_tangent(s)
    ctx.jacobi()
    b = cases.random_state(prob.mesh.num_nodes, prob.N, 62)
    cfg = KrylovConfig(restart=restart, max_iters=400, tolerance=1e-9)
    dev = ctx.gmres(b, cfg)
    monkeypatch.setenv("HBGPU_GMRES_HOST", "1")  # read when a context is created
    ctx2 = gpu_ctx(prob, 0, 0.3)
    ctx2.assemble_tangent(s)
    ctx2.jacobi()
    host = ctx2.gmres(b, cfg)
    assert dev.status == host.status
    assert abs(dev.iterations - host.iterations) <= 1
    assert rel(dev.x, host.x) < 1e-7
    n = min(len(dev.history), len(host.history))
    assert n > 1 and np.allclose(dev.history[:n], host.history[:n], rtol=1e-6, atol=1e-14)


def test_gmres_stagnation_zero_operator(gpu):
    """gmres_solve on a zero operator stagnates and returns the best iterate
    with relative residual 1 (test_linalg.cpp:239-247, linalg.cpp:286-289):
    P = 0 and mass = 0 through the C ABI, unit inverse diagonal."""
    from paper_2411_14315_b200.hbgpu import KrylovConfig

    prob = tube_problem(2, traction=False)
    ctx = gpu_ctx(prob)
    n, nnz, N = ctx.state_len, ctx.nnz, prob.N
    ctx.set_pvals(np.zeros(nnz * 8 * N))
    ctx.set_mass(np.zeros(nnz))
    b = np.ones(n)
    res = ctx.gmres(b, KrylovConfig(), inv_diag=np.ones(n))
    assert res.status == 2
    assert abs(res.relative_residual - 1.0) < 1e-12
    assert not res.x.any()
    orc = ob.Restated(prob)
    ref = orc.gmres(np.zeros(nnz * 8 * N), np.zeros(nnz), b, np.ones(n))
    assert ref["status"] == 2 and abs(ref["relative_residual"] - 1.0) < 1e-12


def test_solve_divergence_errors(gpu):
    """DivergenceError exactly where solve_harmonic throws it
    (hb_solver.cpp:165-186): a residual ratio above divergence_ratio, and a
    non-finite residual; the partial ConvergenceLog is kept."""
    from paper_2411_14315_b200.hbgpu import DivergenceError, GpuContext, SolverConfig

    prob = cases.config_problem(0, mesh=cases.meshgen.hex_cylinder(0.3, 1.0, 3, 3, 6))
    ctx = GpuContext(prob.mesh)
    ctx.set_basis(prob.modes, prob.period)
    ctx.set_fluid(prob.rho, prob.mu)
    ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
    with pytest.raises(DivergenceError) as ei:
        ctx.solve_harmonic(SolverConfig(divergence_ratio=0.5, max_newton_iters=3))
    # iteration 0 has rel = 1 > 0.5: one log entry, then the throw
    assert ei.value.partial_log_csv.count("\n") == 2
    # a non-finite outlet traction: the residual is not finite while tau is
    # (a NaN velocity would raise domain_error from compute_tau first, as in
    # the reference, assembly.cpp:51-53)
    bad = [(k, np.full(prob.N, np.nan)) for k, _ in prob.neumann]
    ctx.set_bcs(prob.dirichlet_g, bad, prob.backflow_beta)
    with pytest.raises(DivergenceError, match="not finite"):
        ctx.solve_harmonic(SolverConfig(max_newton_iters=3))
    # the context's assembly config is untouched by the failed solves
    ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
    ctx.set_assembly_config(0, 0.3)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.3)
    s = cases.random_state(prob.mesh.num_nodes, prob.N, 9)
    assert rel(ctx.assemble_tangent(s), orc.tangent(s)) < TOL


def test_solve_restores_assembly_config(gpu):
    """solve_harmonic builds its own AssemblyConfig (pseudo_c1 = 1.5, the
    solver's tau mode and pseudo-dt) and restores the caller's afterwards."""
    from paper_2411_14315_b200.hbgpu import SolverConfig

    prob = tube_problem(3, h=0.25, traction=False)
    ctx = gpu_ctx(prob, 1, 0.7)
    ctx.set_assembly_config(1, 0.7, 2.5, False)
    ctx.solve_harmonic(SolverConfig(max_newton_iters=2))
    orc = ob.Restated(prob, tau_mode=1, pseudo_dt=0.7, pseudo_c1=2.5)
    s = cases.random_state(prob.mesh.num_nodes, prob.N, 19)
    assert rel(ctx.assemble_tangent(s), orc.tangent(s)) < TOL


def test_max_modes_and_bcs_validation(gpu):
    """M = 32 (N = 63, the supported maximum) matches the oracle; M = 33 is
    rejected by set_basis; set_bcs with a bad patch index leaves the
    context's boundary data unchanged."""
    from paper_2411_14315_b200 import meshgen

    mesh = meshgen.cube_delaunay(1500, seed=21)
    M = 32
    N = 2 * M - 1
    neu = [(k, np.full(N, 20.0)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    prob = Problem(mesh, M, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 3 * N), neu, 0.2)
    ctx = gpu_ctx(prob, 0, 0.05)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.05)
    s = cases.random_modes_state(mesh.num_nodes, M, 5)
    r0 = ctx.assemble_residual(s)
    assert rel(r0, orc.residual(s)) < TOL
    p = ctx.assemble_tangent(s)
    assert rel(p, orc.tangent(s)) < TOL
    y = cases.random_state(mesh.num_nodes, N, 6)
    assert rel(ctx.matvec(y), orc.matvec(p, orc.mass(), y)) < TOL
    with pytest.raises(ValueError):
        ctx.set_bcs(None, [(len(mesh.patches) + 1, np.zeros(N))], 0.2)
    assert np.array_equal(ctx.assemble_residual(s), r0)
    with pytest.raises(ValueError):
        ctx.set_basis(33, 1.0)


def test_gmres_generic_host_operator(gpu):
    """The generic gmres_solve(apply, rhs, inv_diag, cfg) overload
    (linalg.hpp:107-109) through hbgpu_gmres_apply: the zero operator of
    test_linalg.cpp:239-247 (n = 8) stagnates with relative residual 1, and the
    restated tangent operator as a host callback converges to the same
    solution and iteration count as the device operator."""
    from paper_2411_14315_b200.hbgpu import KrylovConfig

    prob = tube_problem(3, h=0.25, traction=False)
    ctx = gpu_ctx(prob, 0, 0.3)
    res0 = ctx.gmres_apply(lambda y: np.zeros_like(y), np.ones(8), np.ones(8))
    assert res0.status == 2 and abs(res0.relative_residual - 1.0) < 1e-12
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.3)
    s = cases.random_state(prob.mesh.num_nodes, prob.N, 61, 0.5)
    p = ctx.assemble_tangent(s)
    m = orc.mass()
    inv, _ = ctx.jacobi()
    b = cases.random_state(prob.mesh.num_nodes, prob.N, 62)
    cfg = KrylovConfig(restart=60, max_iters=2000, tolerance=1e-9)
    dev = ctx.gmres(b, cfg)
    host = ctx.gmres_apply(lambda y: orc.matvec(p, m, y), b, inv, cfg)
    assert dev.status == 0 and host.status == 0
    assert abs(dev.iterations - host.iterations) <= 2
    assert rel(host.x, dev.x) < 1e-6
    scale = np.sqrt(np.abs(inv))
    rr = np.linalg.norm(scale * (b - orc.matvec(p, m, host.x))) / np.linalg.norm(scale * b)
    assert rr <= 1e-9 * 1.0001
