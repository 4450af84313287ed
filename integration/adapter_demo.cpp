// adapter_demo — the reference's own case plumbing driving both the reference
// hot path and the GPU adapter (hbflow::gpu::*) on identical inputs.
// Test infrastructure: links the compiled reference (oracle/_ref/libhbref.so)
// for build_case / generate_tube / the CPU functions, and libhbgpu.so.
// Prints one JSON line; exit code 0 iff every parity bound holds.
#include "hbflow_gpu.hpp"

#include "hbflow/cases.hpp"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>

using namespace hbflow;

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0.0, den = 0.0;
    for (size_t k = 0; k < a.size(); ++k) {
        num += (a[k] - b[k]) * (a[k] - b[k]);
        den += b[k] * b[k];
    }
    return std::sqrt(num / (den > 0 ? den : 1.0));
}

int main() {
    CaseDefinition def;
    def.mesh_kind = "tube";
    def.tube_radius = 0.3;
    def.tube_length = 1.5;
    def.mesh_h = 0.15;
    def.modes = 3;
    def.mean_flow = 2.0;
    def.outlet_pressure_mmhg = 10.0;
    CaseInputs in = build_case(def);
    const Mesh& mesh = in.mesh;
    const auto geoms = precompute_geometry(mesh);
    SpectralOperators ops(in.basis);
    const int N = in.basis.time_points;

    HarmonicState state(in.basis, mesh.num_nodes());
    std::mt19937 rng(7);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (auto& v : state.data)
        v = dist(rng);
    AssemblyConfig acfg;
    acfg.pseudo_dt = 0.05;

    const auto r_ref = assemble_residual(mesh, geoms, state, ops, in.props, in.bcs, acfg, 4);
    const auto r_gpu = gpu::assemble_residual(mesh, geoms, state, ops, in.props, in.bcs, acfg);
    const double e_res = rel(r_gpu, r_ref);

    auto pattern = std::make_shared<NodePattern>(NodePattern::build(mesh));
    TangentOperator L;
    L.mesh = &mesh;
    L.ops = &ops;
    L.pattern = pattern;
    L.P = BlockSparseMatrix(pattern, N);
    L.mass = assemble_mass(mesh, geoms, in.props.rho, *pattern);
    BlockSparseMatrix Pg(pattern, N);
    assemble_tangent(mesh, geoms, state, in.props, in.bcs, acfg, L.P);
    gpu::assemble_tangent(mesh, geoms, state, in.props, in.bcs, acfg, Pg);
    const double e_tan = rel(Pg.vals, L.P.vals);
    const auto mass_g = gpu::assemble_mass(mesh, geoms, in.props.rho, *pattern);
    const double e_mass = rel(mass_g, L.mass);

    std::vector<double> y(L.size()), o_ref(L.size()), o_gpu(L.size());
    for (auto& v : y)
        v = dist(rng);
    L.matvec(y, o_ref);
    gpu::matvec(L, y, o_gpu);
    const double e_mv = rel(o_gpu, o_ref);

    // in-place edits of host data the adapter has already mirrored on the
    // device must be seen (content fingerprints, not pointer identity)
    for (size_t k = 0; k < L.P.vals.size(); k += 3)
        L.P.vals[k] *= 1.25;
    for (auto& m : L.mass)
        m *= 0.75;
    L.matvec(y, o_ref);
    gpu::matvec(L, y, o_gpu);
    const double e_inplace_op = rel(o_gpu, o_ref);
    // ramped Dirichlet data edited in place (same vector): dirichlet_g enters
    // through install_dirichlet in solve_harmonic (assembly.cpp:429-441)
    BoundaryConditionSet bcs2 = in.bcs;
    SolverConfig ramp;
    ramp.max_newton_iters = 2;
    ramp.krylov.tolerance = 1e-12;
    ramp.krylov.max_iters = 4000;
    const auto r_gpu2a = gpu::solve_harmonic(mesh, geoms, in.basis, in.props, bcs2, ramp);
    for (auto& g : bcs2.dirichlet_g)
        g *= 0.5;
    const auto s_ref2 = solve_harmonic(mesh, geoms, in.basis, in.props, bcs2, ramp);
    const auto s_gpu2 = gpu::solve_harmonic(mesh, geoms, in.basis, in.props, bcs2, ramp);
    const double e_inplace_g = rel(s_gpu2.state.data, s_ref2.state.data);
    const double d_g = rel(r_gpu2a.state.data, s_ref2.state.data);  // the edit is visible
    assemble_tangent(mesh, geoms, state, in.props, in.bcs, acfg, L.P);  // restore P
    L.mass = assemble_mass(mesh, geoms, in.props.rho, *pattern);

    const auto pc_ref = jacobi_preconditioner(L);
    const auto pc_gpu = gpu::jacobi_preconditioner(L);
    const double e_jac = rel(pc_gpu.inv_diag, pc_ref.inv_diag);
    KrylovConfig kc;
    kc.tolerance = 1e-8;
    const auto lin = gpu::gmres_solve(L, r_ref, pc_gpu, kc);
    std::vector<double> Lx(L.size()), sres(L.size()), sb(L.size());
    L.matvec(lin.x, Lx);
    for (size_t k = 0; k < L.size(); ++k) {
        const double s = std::sqrt(std::abs(pc_ref.inv_diag[k]));
        sres[k] = s * (r_ref[k] - Lx[k]);
        sb[k] = s * r_ref[k];
    }
    std::vector<double> zero(L.size(), 0.0);
    const double gmres_scaled = rel(sres, zero) / rel(sb, zero);

    // the generic gmres_solve overload (linalg.hpp:107-109) with a lambda:
    // the reference's zero-operator stagnation case (test_linalg.cpp:239-247)
    // and the tangent operator as a lambda, against the reference's generic GMRES
    const std::function<void(std::span<const double>, std::span<double>)> zero_op =
        [](std::span<const double>, std::span<double> out) { std::fill(out.begin(), out.end(), 0.0); };
    std::vector<double> b8(8, 1.0), ones8(8, 1.0);
    const auto g_zero = gpu::gmres_solve(zero_op, b8, ones8, KrylovConfig{});
    const bool zero_ok = g_zero.status == KrylovStatus::Stagnated && std::abs(g_zero.relative_residual - 1.0) < 1e-12;
    const std::function<void(std::span<const double>, std::span<double>)> Lop =
        [&L](std::span<const double> y, std::span<double> out) { L.matvec(y, out); };
    KrylovConfig kc2;
    kc2.tolerance = 1e-9;
    kc2.restart = 60;
    kc2.max_iters = 3000;
    const auto g_lam = gpu::gmres_solve(Lop, r_ref, pc_ref.inv_diag, kc2);
    const auto r_lam = gmres_solve(Lop, r_ref, pc_ref.inv_diag, kc2);
    const double e_lambda = rel(g_lam.x, r_lam.x);
    const bool lambda_ok = g_lam.status == KrylovStatus::Converged && r_lam.status == KrylovStatus::Converged &&
                           e_lambda < 1e-6 &&
                           std::abs(g_lam.iterations - r_lam.iterations) <= std::max(3, r_lam.iterations / 10);

    SolverConfig scfg;
    scfg.newton_tol_orders = 10.0;
    scfg.max_newton_iters = 300;
    scfg.krylov.tolerance = 1e-10;
    scfg.krylov.max_iters = 5000;
    scfg.pseudo_dt = 3.0 * suggest_pseudo_dt(mesh, in.bcs, in.basis).dt;
    auto t0 = std::chrono::steady_clock::now();
    const auto s_ref = solve_harmonic(mesh, geoms, in.basis, in.props, in.bcs, scfg);
    auto t1 = std::chrono::steady_clock::now();
    const auto s_gpu = gpu::solve_harmonic(mesh, geoms, in.basis, in.props, in.bcs, scfg);
    auto t2 = std::chrono::steady_clock::now();
    const double e_solve = rel(s_gpu.state.data, s_ref.state.data);

    // time-stepping solver (time_solver.cpp) on the same case plumbing
    TimeSolverConfig tcfg = TimeSolverConfig::from_case(def);
    tcfg.steps_per_cycle = 40;
    tcfg.cycles = 2;
    auto t3 = std::chrono::steady_clock::now();
    const auto ts_ref = solve_time(in, tcfg);
    auto t4 = std::chrono::steady_clock::now();
    const auto ts_gpu = gpu::solve_time(in, tcfg);
    auto t5 = std::chrono::steady_clock::now();
    const double e_time_u = rel(ts_gpu.cycle.u, ts_ref.cycle.u);
    const double e_time_p = rel(ts_gpu.cycle.p, ts_ref.cycle.p);

    const bool ok = zero_ok && lambda_ok && e_inplace_op < 1e-12 && e_inplace_g < 1e-8 && d_g > 1e-3 &&
                    e_res < 1e-12 && e_tan < 1e-12 && e_mass < 1e-15 && e_mv < 1e-12 &&
                    e_jac < 1e-15 && gmres_scaled <= 1e-8 * 1.0001 && s_ref.log.converged &&
                    s_gpu.log.converged && e_solve < 1e-8 && e_time_u < 1e-8 && e_time_p < 1e-8 &&
                    ts_gpu.total_steps == ts_ref.total_steps;
    std::printf(
        "{\"elements\": %d, \"N\": %d, \"residual\": %.3e, \"tangent\": %.3e, \"mass\": %.3e, "
        "\"matvec\": %.3e, \"jacobi\": %.3e, \"gmres_scaled_residual\": %.3e, \"gmres_iters\": %d, "
        "\"solve_state\": %.3e, \"newton_ref\": %zu, \"newton_gpu\": %zu, \"solve_ref_s\": %.3f, "
        "\"solve_gpu_s\": %.3f, \"time_u\": %.3e, \"time_p\": %.3e, \"time_newton_ref\": %d, "
        "\"time_newton_gpu\": %d, \"time_ref_s\": %.3f, \"time_gpu_s\": %.3f, "
        "\"inplace_operator\": %.3e, \"inplace_dirichlet\": %.3e, \"generic_gmres_zero_stagnated\": %s, "
        "\"generic_gmres_lambda\": %.3e, \"generic_gmres_iters\": [%d, %d], \"ok\": %s}\n",
        mesh.num_elements(), N, e_res, e_tan, e_mass, e_mv, e_jac, gmres_scaled, lin.iterations,
        e_solve, s_ref.log.entries.size(), s_gpu.log.entries.size(),
        std::chrono::duration<double>(t1 - t0).count(),
        std::chrono::duration<double>(t2 - t1).count(), e_time_u, e_time_p, ts_ref.total_newton_iters,
        ts_gpu.total_newton_iters, std::chrono::duration<double>(t4 - t3).count(),
        std::chrono::duration<double>(t5 - t4).count(), e_inplace_op, e_inplace_g, zero_ok ? "true" : "false",
        e_lambda, g_lam.iterations, r_lam.iterations, ok ? "true" : "false");
    gpu::release(mesh);
    return ok ? 0 : 1;
}
