/* hbgpu.h — C ABI of the B200-native HB-GLS hot path (libhbgpu.so).
 *
 * Drop-in boundary for the reference solver's hot-path calls
 * (reference = /root/reference/proj, C++20 CPU code).  Each entry point names
 * the reference interface it replaces.  A C++ adapter with the reference's
 * exact signatures forwards to these functions, so
 * solve_harmonic (src/hb_solver.cpp:113-221) is the only call-site change.
 *
 * Conventions
 *  - Plain pointers and sizes; no C++ or torch types.  Host buffers unless a
 *    function name ends in _dev (device pointers, ordered on the context's
 *    CUDA stream, see hbgpu_stream()).
 *  - Layouts are the reference's:
 *      state / residual   (node*4 + comp)*N + n, comp 3 = pressure  (assembly.hpp:25-47)
 *      dirichlet_g        (node*3 + i)*N + n                         (assembly.hpp:52-54)
 *      geometry           22 doubles per element = ElementGeometry  (mesh.hpp:26-34)
 *      BSR values         (blk*8 + slot)*N + n, slots K|G1..3|D1..3|L (linalg.hpp:30-51)
 *      pattern            CSR row_ptr[nn+1], col_idx[nnz], sorted    (linalg.hpp:14-23)
 *  - Every function returns an hbgpu_status; the adapter rethrows the
 *    matching reference exception (errors.hpp, std::invalid_argument,
 *    std::domain_error).  hbgpu_last_error() gives the message.
 *  - A context is not thread-safe (one solve owns it); the
 *    reference's `threads` arguments have no GPU meaning and are not taken.
 *  - No CPU fallback: creating a context without a usable sm_100 device fails
 *    with HBGPU_ERR_CUDA.
 */
#ifndef HBGPU_H
#define HBGPU_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HBGPU_OK = 0,
    HBGPU_ERR_INVALID = 1,     /* std::invalid_argument (linalg.cpp:45-46,81-82) */
    HBGPU_ERR_DOMAIN = 2,      /* std::domain_error, singular tau (assembly.cpp:51-53) */
    HBGPU_ERR_GEOMETRY = 3,    /* GeometryError (mesh.cpp:173-174) */
    HBGPU_ERR_PARSE = 4,       /* ParseError (spectral.cpp:19-22) */
    HBGPU_ERR_STAGNATION = 5,  /* StagnationError (hb_solver.cpp:200-203) */
    HBGPU_ERR_DIVERGENCE = 6,  /* DivergenceError (hb_solver.cpp:165-186) */
    HBGPU_ERR_CUDA = 7,
    HBGPU_ERR_OOM = 8
} hbgpu_status;

typedef struct hbgpu_ctx hbgpu_ctx;

/* Mesh after Mesh::finalize (mesh.cpp:60-157): oriented elements and facets,
 * outward unit normals and facet areas, Dirichlet node mask.  `geometry` may
 * be the reference's std::vector<ElementGeometry>::data() (zero-copy); when
 * NULL it is computed on the device from xyz (element_geometry, mesh.cpp:159-203). */
typedef struct {
    int num_nodes;
    int num_elements;
    const double* xyz;                /* nn*3; may be NULL when geometry is given */
    const int* conn;                  /* ne*4 */
    const double* geometry;           /* ne*22 or NULL */
    const unsigned char* dirichlet;   /* nn, Mesh::is_dirichlet_node */
    int num_patches;
    const int* patch_kind;            /* 0 = Dirichlet, 1 = Neumann */
    const int* patch_num_facets;
    const int* facets;                /* sum(patch_num_facets)*3, patch-major */
    const double* normals;            /* same count * 3 */
    const double* areas;              /* same count */
} hbgpu_mesh_desc;

/* Uploads the mesh, builds NodePattern (linalg.cpp:10-30) and the device
 * incidence structures.  Returns NULL on failure (*status says why). */
hbgpu_ctx* hbgpu_create(const hbgpu_mesh_desc* mesh, int* status);
void hbgpu_destroy(hbgpu_ctx* ctx);
const char* hbgpu_last_error(const hbgpu_ctx* ctx);
/* Message of the last failed hbgpu_create on this thread. */
const char* hbgpu_create_error(void);
/* cudaStream_t of the context, as void*. */
void* hbgpu_stream(hbgpu_ctx* ctx);
int hbgpu_synchronize(hbgpu_ctx* ctx);

/* Largest supported mode count (N = 63 time samples; BASELINE.json's largest is
 * M = 24, the paper's N = 25).  hbgpu_set_basis rejects larger M with
 * HBGPU_ERR_INVALID instead of failing at the first launch. */
#define HBGPU_MAX_MODES 32

/* SpectralBasis(M, T) (spectral.cpp:18-27) + SpectralOperators (H = E^-1 Omega E,
 * spectral.cpp:146-164,236-256), applied as a dense N x N matrix on device. */
int hbgpu_set_basis(hbgpu_ctx* ctx, int modes, double period);
/* FluidProperties (assembly.hpp:17-23); validate() semantics (assembly.cpp:38-41). */
int hbgpu_set_fluid(hbgpu_ctx* ctx, double rho, double mu);
/* BoundaryConditionSet (assembly.hpp:50-60): dirichlet_g nn*3*N (may be NULL =
 * zeros), Neumann list (patch index, h[N] each, h is n_neumann*N), backflow beta. */
int hbgpu_set_bcs(hbgpu_ctx* ctx, const double* dirichlet_g, int n_neumann,
                  const int* neumann_patch, const double* neumann_h, double backflow_beta);
/* AssemblyConfig (assembly.hpp:64-70): tau_mode 0 = QuadraturePoint, 1 = ElementMean;
 * pseudo_dt <= 0 or non-finite = infinity (no pseudo-time term). */
int hbgpu_set_assembly_config(hbgpu_ctx* ctx, int tau_mode, double pseudo_dt, double pseudo_c1,
                              int backflow_in_tangent);

/* Sizes: nodes, elements, time points N, pattern nnz, state length nn*4*N. */
int hbgpu_sizes(const hbgpu_ctx* ctx, int* num_nodes, int* num_elements, int* time_points,
                long long* nnz, long long* state_len);
/* NodePattern export (bit-exact target vs linalg.cpp:10-30). */
int hbgpu_get_pattern(hbgpu_ctx* ctx, int* row_ptr, int* col_idx);
/* Device-computed ElementGeometry (22 doubles per element). */
int hbgpu_get_geometry(hbgpu_ctx* ctx, double* geometry);

/* ---- drop-ins (host buffers) ------------------------------------------ */

/* assemble_residual (assembly.hpp:129-134, assembly.cpp:443-548). */
int hbgpu_assemble_residual(hbgpu_ctx* ctx, const double* state, double* residual);
/* One Newton iteration's assembly of a host state: assemble_residual (into
 * the host `residual`) and assemble_tangent (P kept on the device for the
 * following matvec / jacobi / gmres calls) of the same state — the pair of
 * calls at hb_solver.cpp:152,161 with a single upload; the residual's copy back
 * overlaps the tangent. */
int hbgpu_assemble(hbgpu_ctx* ctx, const double* state, double* residual);
/* assemble_tangent (assembly.hpp:138-141, assembly.cpp:550-666).  P stays on
 * the device for hbgpu_matvec / hbgpu_jacobi / hbgpu_gmres; pvals may be NULL. */
int hbgpu_assemble_tangent(hbgpu_ctx* ctx, const double* state, double* pvals);
/* assemble_mass (assembly.hpp:145-146, assembly.cpp:668-681).  Kept on device; mass may be NULL. */
int hbgpu_assemble_mass(hbgpu_ctx* ctx, double* mass);
/* Replace the device node-pair mass (TangentOperator::mass, nnz doubles). */
int hbgpu_set_mass(hbgpu_ctx* ctx, const double* mass);
/* Replace the device P values (e.g. a P assembled elsewhere), nnz*8*N doubles. */
int hbgpu_set_pvals(hbgpu_ctx* ctx, const double* pvals);
/* TangentOperator::matvec (linalg.hpp:75, linalg.cpp:78-128): out = (P + H (x) mass) y. */
int hbgpu_matvec(hbgpu_ctx* ctx, const double* y, double* out);
/* BlockSparseMatrix::matvec, accumulate = false (linalg.hpp:55-57, linalg.cpp:41-76). */
int hbgpu_bsr_matvec(hbgpu_ctx* ctx, const double* y, double* out);
/* jacobi_preconditioner (linalg.hpp:84, linalg.cpp:130-154).  Stored on device;
 * inv_diag may be NULL. */
int hbgpu_jacobi(hbgpu_ctx* ctx, double* inv_diag, int* degenerate_entries);

typedef struct {
    int restart;       /* KrylovConfig (linalg.hpp:86-90): 200 */
    int max_iters;     /* 1000 */
    double tolerance;  /* 0.03, relative, of the split-scaled system */
} hbgpu_krylov_cfg;

typedef struct {
    int iterations;
    double relative_residual;
    int status;        /* KrylovStatus: 0 Converged, 1 MaxIterations, 2 Stagnated */
    int history_len;   /* entries written to `history` (<= capacity) */
    int reorthogonalizations; /* Arnoldi steps that needed the second Gram-Schmidt pass */
} hbgpu_krylov_result;

/* gmres_solve(TangentOperator, rhs, JacobiPreconditioner, cfg)
 * (linalg.hpp:102-115, linalg.cpp:167-293) with the device operator.
 * inv_diag NULL = the context's current Jacobi vector. */
int hbgpu_gmres(hbgpu_ctx* ctx, const double* rhs, const double* inv_diag,
                const hbgpu_krylov_cfg* cfg, double* x, hbgpu_krylov_result* result,
                double* history, int history_capacity);

/* Host-side linear operator for hbgpu_gmres_apply: out = A y, n doubles each. */
typedef void (*hbgpu_apply_fn)(void* user, const double* y, double* out);

/* gmres_solve(const std::function<void(span<const double>, span<double>)>& apply,
 * rhs, inv_diag, cfg) (linalg.hpp:107-109, linalg.cpp:167-293): the generic
 * overload, with the operator supplied by the caller on the host.  The Krylov
 * basis, Gram-Schmidt passes, Givens rotations and the restart / stagnation /
 * iteration-cap logic run on the device as in hbgpu_gmres; each operator
 * application copies the vector to the host, calls `apply`, and copies the
 * result back.  n <= the context's state length.  Overwrites the context's
 * Jacobi vector. */
int hbgpu_gmres_apply(hbgpu_ctx* ctx, hbgpu_apply_fn apply, void* user, long long n, const double* rhs,
                      const double* inv_diag, const hbgpu_krylov_cfg* cfg, double* x,
                      hbgpu_krylov_result* result, double* history, int history_capacity);

/* ---- device-resident fast path (device pointers, ctx stream) ----------- */
int hbgpu_assemble_residual_dev(hbgpu_ctx* ctx, const double* d_state, double* d_residual);
int hbgpu_assemble_tangent_dev(hbgpu_ctx* ctx, const double* d_state);
/* Residual + tangent of one state (one Newton iteration's assembly); the two
 * run concurrently on the context's two streams.  Ordered on hbgpu_stream(). */
int hbgpu_assemble_dev(hbgpu_ctx* ctx, const double* d_state, double* d_residual);
int hbgpu_matvec_dev(hbgpu_ctx* ctx, const double* d_y, double* d_out);
int hbgpu_bsr_matvec_dev(hbgpu_ctx* ctx, const double* d_y, double* d_out);
int hbgpu_jacobi_dev(hbgpu_ctx* ctx, int* degenerate_entries);
int hbgpu_gmres_dev(hbgpu_ctx* ctx, const double* d_rhs, const hbgpu_krylov_cfg* cfg,
                    double* d_x, hbgpu_krylov_result* result, double* history,
                    int history_capacity);
/* Resistance outlets (BASELINE config 3: R = 1e4 dyn s/cm^5) — new physics, not in
 * the reference.  Neumann patch `patch[k]` gets the traction
 * -R[k] Q(n) n on top of its Neumann data, Q(n) = outward flux of u(n) through the
 * patch: r_m[A,i,n] += R Q(n) b[A,i] with b[A,i] = sum over A's facets of area/3 n_i,
 * and TangentOperator::matvec gains R b b^T on free velocity rows/columns per
 * sample (BSR matvec and Jacobi unchanged).  R = 0 / n = 0 removes them. */
int hbgpu_set_resistance(hbgpu_ctx* ctx, int n, const int* patch, const double* R);

/* Copy of the context's current P values (BlockSparseMatrix::vals layout), e.g.
 * after hbgpu_assemble, which keeps P on the device. */
int hbgpu_get_pvals(hbgpu_ctx* ctx, double* pvals);

/* Block rows of the context's current P: for each listed node A (distinct or
 * not), the segment vals[row_ptr[A]*8N .. row_ptr[A+1]*8N) appended to `out`
 * in list order (the reference's BlockSparseMatrix::vals layout, 64-bit
 * offsets).  Reads back a sample of P without copying all of it (P is 34.6 GB
 * at BASELINE config 4, Nm = 24). */
int hbgpu_get_pvals_rows(hbgpu_ctx* ctx, int nrows, const int* rows, double* out);

/* Device pointers of the context's P values / mass / inverse diagonal. */
double* hbgpu_pvals_dev(hbgpu_ctx* ctx);

/* ---- Newton driver ------------------------------------------------------- */

typedef struct {
    double pseudo_dt;          /* SolverConfig (hb_solver.hpp:12-23): 0 = auto h_c/u_c */
    double newton_tol_orders;  /* 3 */
    int max_newton_iters;      /* 60 */
    hbgpu_krylov_cfg krylov;
    int tau_mode;
    int backflow_in_tangent;
    double divergence_ratio;   /* 1e3 */
} hbgpu_solver_cfg;

typedef struct {
    int entries;               /* ConvergenceLog entries written (<= capacity) */
    int converged;
    double pseudo_dt, cfl;
    double assembly_seconds, linear_seconds, total_seconds;
} hbgpu_solve_info;

/* solve_harmonic (hb_solver.hpp:70-72, hb_solver.cpp:113-221): rest + Dirichlet
 * + outlet pressure start, pseudo-time Newton, device GMRES.  Log arrays have
 * `capacity` entries (iter, res, res_rel, linear_iters, seconds).  state_out
 * receives the final HarmonicState data.  Returns HBGPU_ERR_DIVERGENCE /
 * HBGPU_ERR_STAGNATION exactly where the reference throws. */
int hbgpu_solve_harmonic(hbgpu_ctx* ctx, const hbgpu_solver_cfg* cfg, double* state_out,
                         hbgpu_solve_info* info, int capacity, int* log_iter, double* log_res,
                         double* log_rel, int* log_linear, double* log_seconds);

/* ---- time-domain solver (the paper's comparison baseline) --------------- */

/* TimeDirichletFn (cases.hpp:132-133): g and dg/dt (node*3+i, all nodes) at time t. */
typedef void (*hbgpu_time_dirichlet_fn)(double t, double* g, double* gdot, void* user);

typedef struct {
    int steps_per_cycle;       /* TimeSolverConfig (time_solver.hpp:11-22): 500 */
    int cycles;                /* 4 */
    double rho_inf;            /* 0.2 */
    double newton_tol_orders;  /* 3 */
    int max_newton_iters;      /* 8 */
    hbgpu_krylov_cfg krylov;
    int steady;                /* drop the acceleration term, one steady solve */
    double initial_pressure;   /* initial_pressure_level (assembly.cpp:415-427) of the HB
                                  Neumann data; NaN = from the context's (steady) data */
} hbgpu_time_cfg;

typedef struct {
    double cycle_change;       /* TimeSolution (time_solver.hpp:42-49) */
    double total_seconds;
    int total_steps;
    int total_newton_iters;
    double omega_hat_last;
} hbgpu_time_result;

/* time_residual (time_solver.cpp:58-166) at (u, udot, p) = (node*3+i, node*3+i,
 * node), host buffers; r: node*4+c.  N = 1 context. */
int hbgpu_time_residual(hbgpu_ctx* ctx, const double* u, const double* udot, const double* p,
                        double omega_hat, double* r);
/* time_tangent (time_solver.cpp:172-254) into the context's N = 1 P (kept on
 * the device for hbgpu_matvec / hbgpu_gmres); pvals (nullable) receives it. */
int hbgpu_time_tangent(hbgpu_ctx* ctx, const double* u, double omega_hat, double am, double fg,
                       double* pvals);

/* solve_time (time_solver.hpp:51-54, time_solver.cpp:269-485): generalized-alpha
 * GLS time stepping on the device (time_residual / time_tangent kernels, the
 * N = 1 L-matvec, Jacobi and GMRES).  The context must carry the N = 1 basis
 * (hbgpu_set_basis(ctx, 1, period)); its Neumann values are the steady outlet
 * tractions h[0].  cycle_u / cycle_p (nullable) receive the CycleHistory of
 * the last cycle: (steps+1) x nodes*3 and (steps+1) x nodes snapshots (steady:
 * one snapshot).  HBGPU_ERR_DIVERGENCE / HBGPU_ERR_STAGNATION where the
 * reference throws DivergenceError / StagnationError. */
int hbgpu_solve_time(hbgpu_ctx* ctx, const hbgpu_time_cfg* cfg, double period,
                     hbgpu_time_dirichlet_fn dirichlet, void* user, double* cycle_u,
                     double* cycle_p, hbgpu_time_result* result);

/* ---- measurement ------------------------------------------------------- */

/* Per-phase CUDA-event timing on the context stream (reset on enable).
 * Phases: 0 residual (all), 1 nodal H*u pass, 2 residual element kernels,
 * 3 residual finalize (H*s, boundary, Dirichlet), 4 tangent, 5 L-matvec,
 * 6 Jacobi, 7 GMRES (all), 8 mass. */
int hbgpu_profile_enable(hbgpu_ctx* ctx, int on);
int hbgpu_profile_read(hbgpu_ctx* ctx, int num_phases, double* ms, int* count);
/* Kernel launches issued by the library since load (process-wide). */
long long hbgpu_kernel_launches(void);
/* Measured dense FP64 FMA throughput of the current device (DFMA loop). */
int hbgpu_fp64_peak(double* tflops);

#ifdef __cplusplus
}
#endif

#endif
