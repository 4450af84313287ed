// C-ABI test harness around the COMPILED REFERENCE (/root/reference/proj).
//
// TEST INFRASTRUCTURE ONLY.  This file is mine; it contains no reference
// code.  It is compiled together with the reference's own sources (built in
// place from /root/reference by oracle/Makefile into oracle/_ref/libhbref.so)
// so that tests/, smoke() and bench.py's CPU-baseline leg can call the
// reference implementation of the hot path on identical inputs:
//   assemble_residual   assembly.cpp:443-548
//   assemble_tangent    assembly.cpp:550-666
//   assemble_mass       assembly.cpp:668-681
//   NodePattern::build  linalg.cpp:10-30
//   TangentOperator::matvec, BlockSparseMatrix::matvec  linalg.cpp:41-128
//   jacobi_preconditioner linalg.cpp:130-154
//   gmres_solve         linalg.cpp:167-293
//   solve_harmonic      hb_solver.cpp:113-221
//   solve_time          time_solver.cpp:269-485 (the paper's time-stepping baseline)
// plus the reference's independent test oracles (tests/oracles.cpp).
// The product path (paper_2411_14315_b200/) never links or loads this.

#include "hbflow/assembly.hpp"
#include "hbflow/errors.hpp"
#include "hbflow/hb_solver.hpp"
#include "hbflow/linalg.hpp"
#include "hbflow/mesh.hpp"
#include "hbflow/spectral.hpp"
#include "hbflow/time_solver.hpp"
#include "hbflow/cases.hpp"
#include "oracles.hpp"

#include <cmath>
#include <cstring>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

using namespace hbflow;

namespace {

thread_local std::string g_err;

enum Status {
    kOk = 0,
    kInvalid = 1,
    kDomain = 2,
    kGeometry = 3,
    kParse = 4,
    kStagnation = 5,
    kDivergence = 6,
    kOther = 9,
};

template <typename F>
int guard(F&& f) {
    try {
        f();
        return kOk;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return kInvalid;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return kDomain;
    } catch (const GeometryError& e) {
        g_err = e.what();
        return kGeometry;
    } catch (const ParseError& e) {
        g_err = e.what();
        return kParse;
    } catch (const StagnationError& e) {
        g_err = e.what();
        return kStagnation;
    } catch (const DivergenceError& e) {
        g_err = e.what();
        return kDivergence;
    } catch (const std::exception& e) {
        g_err = e.what();
        return kOther;
    }
}

struct RefMesh {
    Mesh mesh;
};

struct RefCtx {
    const Mesh* mesh = nullptr;
    SpectralBasis basis;
    std::unique_ptr<SpectralOperators> ops;
    FluidProperties props;
    BoundaryConditionSet bcs;
    AssemblyConfig cfg;
    std::vector<ElementGeometry> geoms;
    std::shared_ptr<NodePattern> pattern;
    TangentOperator L;
};

} // namespace

extern "C" {

const char* hbref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- meshes

void* hbref_mesh_create(int nn, const double* xyz, int ne, const int* elems, int npatch,
                        const char* names_nl, const int* kinds, const int* nfacets,
                        const int* facets) {
    auto* m = new RefMesh;
    const int st = guard([&] {
        m->mesh.nodes.resize(size_t(nn));
        for (int a = 0; a < nn; ++a)
            m->mesh.nodes[size_t(a)] = {xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]};
        m->mesh.elements.resize(size_t(ne));
        for (int e = 0; e < ne; ++e)
            m->mesh.elements[size_t(e)] = {elems[4 * e], elems[4 * e + 1], elems[4 * e + 2],
                                           elems[4 * e + 3]};
        std::istringstream names(names_nl ? names_nl : "");
        size_t off = 0;
        for (int p = 0; p < npatch; ++p) {
            BoundaryPatch bp;
            std::getline(names, bp.name);
            bp.kind = kinds[p] == 0 ? PatchKind::Dirichlet : PatchKind::Neumann;
            for (int f = 0; f < nfacets[p]; ++f, ++off)
                bp.facets.push_back({facets[3 * off], facets[3 * off + 1], facets[3 * off + 2]});
            m->mesh.patches.push_back(std::move(bp));
        }
        m->mesh.finalize();
    });
    if (st != kOk) {
        delete m;
        return nullptr;
    }
    return m;
}

void* hbref_mesh_tube(double radius, double length, double h) {
    auto* m = new RefMesh;
    if (guard([&] { m->mesh = generate_tube(radius, length, h); }) != kOk) {
        delete m;
        return nullptr;
    }
    return m;
}

void* hbref_mesh_bifurcation(double width, double depth, double inlet_length,
                             double branch_length, double h) {
    auto* m = new RefMesh;
    if (guard([&] {
            m->mesh = generate_bifurcation(width, depth, inlet_length, branch_length, h);
        }) != kOk) {
        delete m;
        return nullptr;
    }
    return m;
}

void hbref_mesh_destroy(void* mh) { delete static_cast<RefMesh*>(mh); }

int hbref_mesh_sizes(void* mh, int* nn, int* ne, int* npatch, int* total_facets) {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    *nn = m.num_nodes();
    *ne = m.num_elements();
    *npatch = int(m.patches.size());
    int tf = 0;
    for (const auto& p : m.patches)
        tf += int(p.facets.size());
    *total_facets = tf;
    return kOk;
}

// Exports the FINALIZED mesh: oriented elements, oriented facets, normals,
// areas, patch kinds and the Dirichlet node mask (mesh.cpp:60-157).
int hbref_mesh_export(void* mh, double* xyz, int* elems, int* kinds, int* nfacets, int* facets,
                      double* normals, double* areas, unsigned char* dirichlet_mask) {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    for (int a = 0; a < m.num_nodes(); ++a)
        for (int i = 0; i < 3; ++i)
            xyz[3 * a + i] = m.nodes[size_t(a)][size_t(i)];
    for (int e = 0; e < m.num_elements(); ++e)
        for (int k = 0; k < 4; ++k)
            elems[4 * e + k] = m.elements[size_t(e)][size_t(k)];
    size_t off = 0;
    for (size_t p = 0; p < m.patches.size(); ++p) {
        const auto& bp = m.patches[p];
        kinds[p] = bp.kind == PatchKind::Dirichlet ? 0 : 1;
        nfacets[p] = int(bp.facets.size());
        for (size_t f = 0; f < bp.facets.size(); ++f, ++off) {
            for (int k = 0; k < 3; ++k) {
                facets[3 * off + k] = bp.facets[f][size_t(k)];
                normals[3 * off + k] = bp.normals[f][size_t(k)];
            }
            areas[off] = bp.facet_areas[f];
        }
    }
    for (int a = 0; a < m.num_nodes(); ++a)
        dirichlet_mask[a] = (unsigned char)(m.is_dirichlet_node[size_t(a)] ? 1 : 0);
    return kOk;
}

int hbref_patch_name(void* mh, int p, char* buf, int len) {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    if (p < 0 || p >= int(m.patches.size()))
        return kInvalid;
    std::snprintf(buf, size_t(len), "%s", m.patches[size_t(p)].name.c_str());
    return kOk;
}

// 22 doubles per element in ElementGeometry's own memory order:
// grad_N[4][3], volume, xi[9] (mesh.hpp:26-34).
int hbref_geometry(void* mh, double* out) {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    return guard([&] {
        static_assert(sizeof(ElementGeometry) == 22 * sizeof(double));
        const auto g = precompute_geometry(m);
        std::memcpy(out, g.data(), g.size() * sizeof(ElementGeometry));
    });
}

double hbref_characteristic_length(void* mh) {
    return characteristic_length(static_cast<RefMesh*>(mh)->mesh);
}

// Pass col_idx = nullptr to query nnz first.
int hbref_pattern(void* mh, int* row_ptr, int* col_idx, int* nnz) {
    const Mesh& m = static_cast<RefMesh*>(mh)->mesh;
    return guard([&] {
        const NodePattern p = NodePattern::build(m);
        *nnz = p.nnz();
        if (row_ptr)
            std::memcpy(row_ptr, p.row_ptr.data(), p.row_ptr.size() * sizeof(int));
        if (col_idx)
            std::memcpy(col_idx, p.col_idx.data(), p.col_idx.size() * sizeof(int));
    });
}

// ---------------------------------------------------------------- spectral

int hbref_h_dense(int modes, double period, double* out) {
    return guard([&] {
        SpectralOperators ops(SpectralBasis(modes, period));
        const auto H = ops.dense();
        std::memcpy(out, H.data(), H.size() * sizeof(double));
    });
}

int hbref_oracle_h_dense(int modes, double period, double* out) {
    return guard([&] {
        const auto H = testing::oracle_h_dense(modes, period);
        std::memcpy(out, H.data(), H.size() * sizeof(double));
    });
}

int hbref_apply_h(int modes, double period, const double* in, double* out, int count) {
    return guard([&] {
        SpectralOperators ops(SpectralBasis(modes, period));
        const size_t N = size_t(ops.size());
        std::vector<double> buf(in, in + N * size_t(count));
        auto ws = ops.make_workspace();
        ops.apply_many(buf, buf, count, *ws);
        std::memcpy(out, buf.data(), buf.size() * sizeof(double));
    });
}

// ---------------------------------------------------------------- solver ctx

void* hbref_ctx_create(void* mh, int modes, double period, double rho, double mu) {
    auto* c = new RefCtx;
    const int st = guard([&] {
        c->mesh = &static_cast<RefMesh*>(mh)->mesh;
        c->basis = SpectralBasis(modes, period);
        c->ops = std::make_unique<SpectralOperators>(c->basis);
        c->props = FluidProperties{rho, mu};
        c->geoms = precompute_geometry(*c->mesh);
        c->pattern = std::make_shared<NodePattern>(NodePattern::build(*c->mesh));
        c->bcs.dirichlet_g.assign(size_t(c->mesh->num_nodes()) * 3 * size_t(c->basis.time_points),
                                  0.0);
        c->L.mesh = c->mesh;
        c->L.ops = c->ops.get();
        c->L.pattern = c->pattern;
        c->L.P = BlockSparseMatrix(c->pattern, c->basis.time_points);
        c->L.mass = assemble_mass(*c->mesh, c->geoms, c->props.rho, *c->pattern);
    });
    if (st != kOk) {
        delete c;
        return nullptr;
    }
    return c;
}

void hbref_ctx_destroy(void* ch) { delete static_cast<RefCtx*>(ch); }

int hbref_ctx_set_bcs(void* ch, const double* dirichlet_g, int n_neumann, const int* patch_idx,
                      const double* h, double beta) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        const size_t N = size_t(c->basis.time_points);
        if (dirichlet_g)
            c->bcs.dirichlet_g.assign(dirichlet_g,
                                      dirichlet_g + size_t(c->mesh->num_nodes()) * 3 * N);
        c->bcs.neumann.clear();
        for (int k = 0; k < n_neumann; ++k) {
            BoundaryConditionSet::NeumannBC nb;
            nb.patch_index = patch_idx[k];
            nb.h.assign(h + size_t(k) * N, h + size_t(k + 1) * N);
            c->bcs.neumann.push_back(std::move(nb));
        }
        c->bcs.backflow_beta = beta;
    });
}

int hbref_ctx_set_cfg(void* ch, int tau_mode, double pseudo_dt, double c1, int backflow_tangent) {
    auto* c = static_cast<RefCtx*>(ch);
    c->cfg.tau_mode = tau_mode == 0 ? TauMode::QuadraturePoint : TauMode::ElementMean;
    c->cfg.pseudo_dt = pseudo_dt > 0.0 ? pseudo_dt : std::numeric_limits<double>::infinity();
    c->cfg.pseudo_c1 = c1;
    c->cfg.backflow_in_tangent = backflow_tangent != 0;
    return kOk;
}

static HarmonicState make_state(const RefCtx* c, const double* s) {
    HarmonicState st(c->basis, c->mesh->num_nodes());
    std::memcpy(st.data.data(), s, st.data.size() * sizeof(double));
    return st;
}

int hbref_residual(void* ch, const double* state, int threads, double* r_out) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        const auto st = make_state(c, state);
        const auto r = assemble_residual(*c->mesh, c->geoms, st, *c->ops, c->props, c->bcs,
                                         c->cfg, threads);
        std::memcpy(r_out, r.data(), r.size() * sizeof(double));
    });
}

int hbref_oracle_residual(void* ch, const double* state, double* r_out) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        const auto st = make_state(c, state);
        const auto r = testing::oracle_residual(*c->mesh, st, c->props, c->bcs, c->cfg);
        std::memcpy(r_out, r.data(), r.size() * sizeof(double));
    });
}

int hbref_frozen_residual(void* ch, const double* state, const double* coeff_state,
                          double* r_out) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        const auto st = make_state(c, state);
        const auto cs = make_state(c, coeff_state);
        const auto r = testing::oracle_frozen_residual(*c->mesh, st, cs, c->props, c->cfg);
        std::memcpy(r_out, r.data(), r.size() * sizeof(double));
    });
}

int hbref_tangent(void* ch, const double* state, double* pvals_out) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        const auto st = make_state(c, state);
        assemble_tangent(*c->mesh, c->geoms, st, c->props, c->bcs, c->cfg, c->L.P);
        if (pvals_out)
            std::memcpy(pvals_out, c->L.P.vals.data(), c->L.P.vals.size() * sizeof(double));
    });
}

long long hbref_pvals_size(void* ch) {
    return (long long)static_cast<RefCtx*>(ch)->L.P.vals.size();
}

int hbref_set_pvals(void* ch, const double* pvals) {
    auto* c = static_cast<RefCtx*>(ch);
    std::memcpy(c->L.P.vals.data(), pvals, c->L.P.vals.size() * sizeof(double));
    return kOk;
}

int hbref_mass(void* ch, double* mass_out) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        c->L.mass = assemble_mass(*c->mesh, c->geoms, c->props.rho, *c->pattern);
        std::memcpy(mass_out, c->L.mass.data(), c->L.mass.size() * sizeof(double));
    });
}

int hbref_matvec(void* ch, const double* y, double* out, int threads) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        c->L.threads = threads;
        const size_t n = c->L.size();
        c->L.matvec({y, n}, {out, n});
    });
}

int hbref_bsr_matvec(void* ch, const double* y, double* out, int threads) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        const size_t n = c->L.size();
        c->L.P.matvec({y, n}, {out, n}, threads, false);
    });
}

int hbref_jacobi(void* ch, double* inv_diag, int* degenerate) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        const auto pc = jacobi_preconditioner(c->L);
        std::memcpy(inv_diag, pc.inv_diag.data(), pc.inv_diag.size() * sizeof(double));
        *degenerate = pc.degenerate_entries;
    });
}

int hbref_gmres(void* ch, const double* rhs, const double* inv_diag, int restart, int max_iters,
                double tol, int threads, double* x, int* iters, double* relres, int* status,
                double* hist, int hist_cap, int* hist_len) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        c->L.threads = threads;
        const size_t n = c->L.size();
        KrylovConfig kc;
        kc.restart = restart;
        kc.max_iters = max_iters;
        kc.tolerance = tol;
        const auto res = gmres_solve(
            [c](std::span<const double> y, std::span<double> o) { c->L.matvec(y, o); },
            {rhs, n}, {inv_diag, n}, kc);
        std::memcpy(x, res.x.data(), n * sizeof(double));
        *iters = res.iterations;
        *relres = res.relative_residual;
        *status = int(res.status);
        const int hl = int(res.history.size());
        *hist_len = hl;
        for (int k = 0; k < hl && k < hist_cap; ++k)
            hist[k] = res.history[size_t(k)];
    });
}

int hbref_install_dirichlet(void* ch, double* state) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        auto st = make_state(c, state);
        install_dirichlet(*c->mesh, c->bcs, st);
        std::memcpy(state, st.data.data(), st.data.size() * sizeof(double));
    });
}

double hbref_initial_pressure(void* ch) {
    auto* c = static_cast<RefCtx*>(ch);
    return initial_pressure_level(*c->mesh, c->bcs);
}

double hbref_suggest_pseudo_dt(void* ch) {
    auto* c = static_cast<RefCtx*>(ch);
    return suggest_pseudo_dt(*c->mesh, c->bcs, c->basis).dt;
}

int hbref_dense_tangent(void* ch, const double* state, double* out) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        const auto st = make_state(c, state);
        const auto d =
            testing::oracle_dense_tangent(*c->mesh, c->geoms, st, c->props, c->bcs, c->cfg);
        std::memcpy(out, d.data(), d.size() * sizeof(double));
    });
}

// Full reference Newton solve (hb_solver.cpp:113-221).  Log arrays have
// capacity `cap`; *log_len receives the number of entries.
int hbref_solve(void* ch, double pseudo_dt, double orders, int max_newton, int restart,
                int max_iters, double tol, int tau_mode, int threads, double* state_out,
                int* converged, int cap, int* log_len, double* log_res, double* log_rel,
                int* log_lin, double* out_scalars /* pseudo_dt, cfl, asm_s, lin_s, total_s */) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        SolverConfig cfg;
        cfg.pseudo_dt = pseudo_dt;
        cfg.newton_tol_orders = orders;
        cfg.max_newton_iters = max_newton;
        cfg.krylov.restart = restart;
        cfg.krylov.max_iters = max_iters;
        cfg.krylov.tolerance = tol;
        cfg.tau_mode = tau_mode == 0 ? TauMode::QuadraturePoint : TauMode::ElementMean;
        cfg.threads = threads;
        const auto sol = solve_harmonic(*c->mesh, c->geoms, c->basis, c->props, c->bcs, cfg);
        std::memcpy(state_out, sol.state.data.data(), sol.state.data.size() * sizeof(double));
        *converged = sol.log.converged ? 1 : 0;
        const int n = int(sol.log.entries.size());
        *log_len = n;
        for (int k = 0; k < n && k < cap; ++k) {
            log_res[k] = sol.log.entries[size_t(k)].res;
            log_rel[k] = sol.log.entries[size_t(k)].res_rel;
            log_lin[k] = sol.log.entries[size_t(k)].linear_iters;
        }
        out_scalars[0] = sol.pseudo_dt;
        out_scalars[1] = sol.cfl;
        out_scalars[2] = sol.assembly_seconds;
        out_scalars[3] = sol.linear_seconds;
        out_scalars[4] = sol.total_seconds;
    });
}

// Reference time-stepping solve (time_solver.cpp:269-485) on the context's
// mesh, fluid and boundary data (Neumann h[0] = steady outlet traction), with
// the Dirichlet data g(t), dg/dt(t) from a C callback (TimeDirichletFn).
// out_scalars: cycle_change, total_seconds, omega_hat_last, total_steps,
// total_newton_iters.
typedef void (*hbref_time_dirichlet_fn)(double t, double* g, double* gdot, void* user);
int hbref_solve_time(void* ch, double period, int steps, int cycles, double rho_inf, double orders,
                     int max_newton, int restart, int max_iters, double tol, int steady, int threads,
                     hbref_time_dirichlet_fn fn, void* user, double* cycle_u, double* cycle_p,
                     double* out_scalars) {
    auto* c = static_cast<RefCtx*>(ch);
    return guard([&] {
        CaseInputs in;
        in.def.period = period;
        in.mesh = *c->mesh;
        in.props = c->props;
        in.basis = c->basis;
        in.bcs = c->bcs;
        in.time_dirichlet = [fn, user](double t, std::vector<double>& g, std::vector<double>& gd) {
            fn(t, g.data(), gd.data(), user);
        };
        TimeSolverConfig tc;
        tc.steps_per_cycle = steps;
        tc.cycles = cycles;
        tc.rho_inf = rho_inf;
        tc.newton_tol_orders = orders;
        tc.max_newton_iters = max_newton;
        tc.krylov.restart = restart;
        tc.krylov.max_iters = max_iters;
        tc.krylov.tolerance = tol;
        tc.steady = steady != 0;
        tc.threads = threads;
        const auto sol = solve_time(in, tc);
        if (cycle_u)
            std::memcpy(cycle_u, sol.cycle.u.data(), sol.cycle.u.size() * sizeof(double));
        if (cycle_p)
            std::memcpy(cycle_p, sol.cycle.p.data(), sol.cycle.p.size() * sizeof(double));
        out_scalars[0] = sol.cycle_change;
        out_scalars[1] = sol.total_seconds;
        out_scalars[2] = sol.omega_hat_last;
        out_scalars[3] = double(sol.total_steps);
        out_scalars[4] = double(sol.total_newton_iters);
    });
}

} // extern "C"
