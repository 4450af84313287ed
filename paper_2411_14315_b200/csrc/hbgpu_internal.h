// Internal definitions shared by the kernels (hbgpu_kernels.cu) and the host
// runtime / C ABI (hbgpu_host.cu).  Not part of the public interface.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

namespace hbgpu {

// 4-point tet Gauss rule (reference assembly.cpp:15-20).
constexpr double kQA = 0.5854101966249684544613761;
constexpr double kQB = 0.1381966011250105151795414;
// Gauss-Seidel block: number of partial sums of the deterministic reductions.
constexpr int kRedBlocks = 592;  // 4 x 148 SMs
constexpr int kRedThreads = 256;
// Residual element chunks: elements per chunk (time samples per tile: residual_tile(N)).
constexpr int kChunkElems = 64;
// Compact tangent geometry record (gradN 12, V, symmetric xi 6, xi:xi).
constexpr int kTGeo = 20;

// Tangent v3: threads per row CTA, contributions per diagonal part.
#ifndef TAN_THREADS
#define TAN_THREADS 128
#endif
constexpr int kTanThreads = TAN_THREADS;
constexpr int kTanPart = 8;

// Build-time tuning knobs of the residual element pass.
#ifndef RES_VOLATILE_LDS
#define RES_VOLATILE_LDS 0
#endif
#ifndef RES_MINB
#define RES_MINB 2
#endif
#ifndef TAN5_MINB
#define TAN5_MINB 4
#endif
#ifndef TAN_PIPE
#define TAN_PIPE 1
#endif
#ifndef TAN_SMEM_KB
#define TAN_SMEM_KB 64
#endif
#ifndef MV_PREFETCH
#define MV_PREFETCH 1
#endif
#ifndef MV_UNROLL
#define MV_UNROLL 2
#endif

// 1/sqrt(x) for x > 0: MUFU seed + two Newton steps, branch-free (the
// library rsqrt carries special-case branches the element kernels never need;
// x <= 0 / NaN is flagged and masked by the callers).  Within a few ulp.  One
// volatile asm block, so the compiler cannot sink it into a branch on the
// caller's select (which would cost a BSSY/BRA pair per quadrature point).
#ifdef __CUDACC__
#ifndef RSQRT_NEWTON
#define RSQRT_NEWTON 3
#endif
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
#if RSQRT_NEWTON == 3
    // one cubic (Halley) step from the 2^-22 hardware seed: e = 1 - x y0^2,
    // y = y0 (1 + e (1/2 + 3/8 e)); relative error ~ e^3 < 2^-60 (5 FP64
    // instructions, against 7 for two Newton steps)
    asm volatile(
        "{\n\t.reg .f64 t, e, p, y0;\n\t"
        "rsqrt.approx.ftz.f64 y0, %1;\n\t"
        "mul.rn.f64 t, %1, y0;\n\t"
        "neg.f64 t, t;\n\t"
        "fma.rn.f64 e, t, y0, 0d3FF0000000000000;\n\t"
        "fma.rn.f64 p, e, 0d3FD8000000000000, 0d3FE0000000000000;\n\t"
        "mul.rn.f64 p, p, e;\n\t"
        "fma.rn.f64 %0, y0, p, y0;\n\t}"
        : "=d"(y)
        : "d"(x));
#elif RSQRT_NEWTON == 1
    asm volatile(
        "{\n\t.reg .f64 h, t, e, y0;\n\t"
        "rsqrt.approx.ftz.f64 y0, %1;\n\t"
        "mul.rn.f64 h, %1, 0d3FE0000000000000;\n\t"
        "mul.rn.f64 t, h, y0;\n\t"
        "neg.f64 t, t;\n\t"
        "fma.rn.f64 e, t, y0, 0d3FE0000000000000;\n\t"
        "fma.rn.f64 %0, y0, e, y0;\n\t}"
        : "=d"(y)
        : "d"(x));
#else
    asm volatile(
        "{\n\t.reg .f64 h, t, e, y0;\n\t"
        "rsqrt.approx.ftz.f64 y0, %1;\n\t"
        "mul.rn.f64 h, %1, 0d3FE0000000000000;\n\t"
        "mul.rn.f64 t, h, y0;\n\t"
        "neg.f64 t, t;\n\t"
        "fma.rn.f64 e, t, y0, 0d3FE0000000000000;\n\t"
        "fma.rn.f64 y0, y0, e, y0;\n\t"
        "mul.rn.f64 t, h, y0;\n\t"
        "neg.f64 t, t;\n\t"
        "fma.rn.f64 e, t, y0, 0d3FE0000000000000;\n\t"
        "fma.rn.f64 %0, y0, e, y0;\n\t}"
        : "=d"(y)
        : "d"(x));
#endif
    return y;
}
// tau = arg^-1/2, or 0 when arg <= 0 / NaN (`bad`, flagged by the caller).
// The argument is sanitised and the result masked by a multiply, so the
// Newton iteration is always executed and never sits behind a branch.
// TAU_UNCHECKED (default): a non-positive argument only happens on a degenerate
// element; the caller raises the context's domain-error flag and every output of
// that call is discarded by the host (the reference throws, assembly.cpp:64-66),
// so the value returned for it is irrelevant and the sanitising select + masking
// multiply (1 DMUL + 4 FSEL per quadrature point) are dropped.
#ifndef TAU_UNCHECKED
#define TAU_UNCHECKED 1
#endif
__device__ __forceinline__ double tau_or_zero(double arg, bool bad) {
#if TAU_UNCHECKED
    (void)bad;
    return rsqrt_nr(arg);
#else
    return rsqrt_nr(bad ? 1.0 : arg) * (bad ? 0.0 : 1.0);
#endif
}

// mbarrier + bulk async copy (cp.async.bulk, the TMA engine's 1-D mode)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
// Bulk prefetch into L2 (the TMA engine's 1-D mode, no shared memory).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}
#endif

// Number of kernel launches issued by this library (bench.py's gpu_launches).
extern std::atomic<long long> g_launches;
cudaError_t run_fp64_peak(int blocks, int threads, int iters, double* out, float* ms);

// ---------------------------------------------------------------- kernel args

// Element-chunk residual: chunk c = elements [c*CE, (c+1)*CE); its distinct
// nodes (sorted) are chunk_nodes[chunk_node_ptr[c] ..]; every (chunk, node)
// pair p owns one partial-sum record of 7N doubles (r_u0..2, r_p, s0..2).
struct ResidualChunkArgs {
    const double* tgeom;         // compact geometry records (kTGeo doubles per element)
    const double* state;
    const double* hu;
    // per chunk, a contiguous "chunk pack" (16-byte aligned):
    //   hdr int4 {nloc, ecount, nb (first pair), 0}, nodes int[nloc],
    //   sptr int[nloc + 1] (chunk-relative slot ranges, element order),
    //   soff u16[4 ecount] (slot -> shared-memory offset (el*29 + a*7) * T),
    //   lconn u32[ecount] (4 x u8 chunk-local node ids)
    const unsigned char* rpack;
    const int* rpack_ptr;        // nchunks + 1, 16-byte units
    int max_rpack;               // bytes
    double* partial;             // pairs * 7N
    int ne, N, max_nloc, nchunks;
    long npairs;
    double rho, mu, nu;
    int tau_mode;
    int* flag;
};

struct TangentArgs {
    const double* tgeom;     // kTGeo doubles / element (compact tangent geometry)
    const double* state;
    const uint8_t* dir;      // per node
    const int* row_ptr;
    const int* inc_ptr;      // per node, into inc_rec
    const int4* inc_rec;     // 2 per incidence: conn[4]; {e | a<<30, cols(4 x u8), dirichlet mask, 0}
    double* pvals;
    int N;
    double rho, mu, nu, pseudo_c;
    int tau_mode;
    int* flag;
    // per block, its contributions (i<<2 | b), i = incidence index within
    // the row, in element order
    const int* col_idx;
    const int* diag_blk;
    const int* contrib_ptr;        // nnz + 1
    const uint16_t* contrib;
    int max_inc;
    int NT;            // time samples per CTA (tile of N)
    int max_blk;       // longest block row of the bucket
    // tangent v5: per-block n-invariant sums and off-diagonal visiting order
    const double* blkc;         // nnz x 8
    const uint8_t* blk_order;   // per row: off-diagonal block offsets, descending count
    const int4* rowdesc;        // per bucket row: {A, i0, ninc, k0}, {nblk, cb, kdiag, 0}
};

// Persistent tangent row pipeline (hbgpu_tangent_pipe.cu): per-row packs.
struct PipeArgs {
    const unsigned char* pack;  // row packs, 16-byte aligned
    const int* pack_ptr;        // nrows + 1, in 16-byte units
    int nrows;
    int max_pack;               // bytes
};

struct MatvecArgs {
    const int* row_ptr;
    const int* col_idx;
    const double* vals;
    const double* mass;
    const uint8_t* dir;
    const double* H;
    const double* y;
    double* out;
    const double* scale;      // optional input scaling (gathered): L (S y)
    const double* scale_out;  // optional output scaling: S L y
    const int* perm;          // optional row order (rows of similar length per CTA)
    const int4* rows;         // optional {A, row_ptr[A], row_ptr[A+1], 0} in perm order
    const int* skip;          // optional device stop flag (GMRES steps past convergence)
    int nn, N, rows_per_cta;
    int with_c;
    int lanes;                // lanes per (row, sample): 0 auto, 1 or 4 (tests)
};

struct BoundaryArgs {
    const int* bnode;       // boundary node ids
    const int* bptr;        // per boundary node, into binc
    const int* binc;        // facet*4 + v
    const int* fac;         // facet nodes (3)
    const double* fnormal;  // 3
    const double* farea;
    const int* fbc;         // Neumann entry of the facet
    const double* h;        // nbc*N
    const uint8_t* dir;
    const double* state;
    double* r;
    int nbnodes, N;
    double rho, beta;
};

// ---------------------------------------------------------------- launchers
// (defined in hbgpu_kernels.cu; all asynchronous on `st`)

void launch_geometry(const double* xyz, const int4* conn, int ne, double* geom, int* flag,
                     cudaStream_t st);
void launch_apply_h_series(const double* H, int N, const double* in, int in_node_stride,
                           double* out, int out_node_stride, int nnodes, cudaStream_t st);
size_t residual_smem_bytes(int max_nloc, int max_rpack, int T);
int residual_tile(int N);
size_t residual_pack_bytes(int nloc, int ecount);
void residual_pack_write(unsigned char* dst, int nloc, int ecount, int nb, const int* nodes,
                         const int* sptr_rel, const uint16_t* soff, const uint32_t* lconn);
void launch_residual_chunks(const ResidualChunkArgs& a, int grid, int T, cudaStream_t st);
cudaError_t configure_residual_smem(size_t bytes, int T);
cudaError_t residual_occupancy(int* blocks_per_sm, size_t smem, int T);
void launch_residual_nodes(const double* H, int N, int nn, const int* npart_ptr, const int* npart,
                           const double* partial, const uint8_t* dir, double* r, int T,
                           long npairs, cudaStream_t st);
void launch_boundary(const BoundaryArgs& a, cudaStream_t st);
// resistance outlets: out[free velocity rows] += (scale) R Q b per (patch, sample)
void launch_resistance(const int* ptr, const int* node, const double* b, const double* R, int npatch,
                       const uint8_t* dir, int N, const double* v, double* out, const double* scale, int free_cols,
                       const int* skip, cudaStream_t st);
void launch_mass_rows(const double* geom, const int* row_ptr, const int* inc_ptr, const int4* rec,
                      double rho, double* mass, int nn, cudaStream_t st);
void launch_tangent_geometry(const double* geom, int ne, double* tg, cudaStream_t st);
size_t tangent_row_smem(int max_inc, int max_blk, int max_dparts, int NT);
void launch_tangent_blockconst(const double* tgeom, const int* row_ptr, const int* inc_ptr,
                               const int4* inc_rec, const int* contrib_ptr, const uint16_t* contrib,
                               int nn, double* blkc, cudaStream_t st);
cudaError_t configure_tangent_row_smem(size_t bytes);
void launch_tangent_row(const TangentArgs& a, int nrows, size_t smem, cudaStream_t st);
size_t tangent_pack_bytes(int ninc, int nblk);
void tangent_pack_write(unsigned char* dst, int A, int k0, int ninc, int nblk, int kdiag,
                        const int* cols, const int2* inc, const uint16_t* cont, const int* cptr,
                        const uint8_t* order);
void launch_tangent_pack_refresh(unsigned char* pack, const int* pack_ptr, int nrows,
                                 const uint8_t* dir, const double* blkc, cudaStream_t st);
size_t tangent_pipe_smem(int max_pack, int max_inc, int max_blk, int N, int NT);
cudaError_t configure_tangent_pipe_smem(int threads, size_t bytes);
cudaError_t tangent_pipe_occupancy(int threads, int* blocks_per_sm, size_t smem);
void launch_tangent_pipe(const TangentArgs& a, const PipeArgs& p, int threads, int grid_x, size_t smem,
                         cudaStream_t st);
void launch_backflow_tangent(const BoundaryArgs& a, const int* row_ptr, const int* col_idx,
                             double* pvals, cudaStream_t st);
void launch_lmatvec(const MatvecArgs& a, cudaStream_t st);
void launch_mask_mass(const double* mass, const int* row_ptr, const int* col_idx,
                      const uint8_t* dir, int nn, double* mass_c, cudaStream_t st);
void launch_jacobi(const double* vals, const int* diag_blk, int nn, int N, double* inv_diag,
                   int* degenerate, cudaStream_t st);
void launch_install_dirichlet(const double* g, const uint8_t* dir, int nn, int N, double* state,
                              cudaStream_t st);
void launch_fill_pressure(double p0, int nn, int N, double* state, cudaStream_t st);
void launch_newton_update(const double* dx, const uint8_t* dir, int nn, int N, double* state,
                          cudaStream_t st);

// time-domain operators (hbgpu_time.cu; reference src/time_solver.cpp)
void launch_time_residual(const double* geom, const int4* conn, int ne, const int* inc_ptr, const int4* rec,
                          const uint8_t* dir, int nn, const double* u, const double* udot, const double* p,
                          double rho, double mu, double omega_hat, double* elem, double* r, cudaStream_t st);
void launch_time_tangent(const double* geom, const int* row_ptr, const int* col_idx, const int* inc_ptr,
                         const int4* rec, const uint8_t* dir, int nn, const double* u, double rho, double mu,
                         double omega_hat, double am, double fg, double* vals, cudaStream_t st);
void launch_time_predict(const double* u, const double* ud, const double* p, const double* g, const double* gd,
                         const uint8_t* dir, int nn, int steady, double gamma, double dt, double* nu_, double* nud,
                         double* np, cudaStream_t st);
void launch_time_alpha(const double* u, const double* ud, const double* nu_, const double* nud, int nn,
                       double af, double am, double* ual, double* aal, cudaStream_t st);
void launch_time_update(const double* x, const uint8_t* dir, int nn, int steady, double gdt, double* nu_,
                        double* nud, double* np, cudaStream_t st);
void launch_time_pack(const double* u, const double* p, int nn, double* s4, cudaStream_t st);
void launch_time_wnorm(const double* w, const double* f0, const double* f1, int nn, double* partial,
                       cudaStream_t st);
void launch_time_cycle(const double* f, double* buf, long n3, int accumulate, double* partial, cudaStream_t st);
void launch_nodal_volumes(const double* geom, const int* inc_ptr, const int4* rec, int nn, double* w,
                          cudaStream_t st);

// vectors (length n), deterministic reductions
void launch_sqrt_abs(const double* in, double* out, long n, cudaStream_t st);
void launch_mul(const double* a, const double* b, double* out, long n, cudaStream_t st);
void launch_scaled_diff(const double* s, const double* a, const double* b, double* out, long n,
                        cudaStream_t st);  // out = s*(a-b)
// partial[i*kRedBlocks + b] = block b's share of <V_i, w>, i < nv.
void launch_multidot(const double* V, long ld, int nv, const double* w, long n, double* partial,
                     cudaStream_t st);
// out[i] = sum_b partial[i*kRedBlocks+b] (fixed order); optional sqrt of out[0]
// `skip` (nullable, device): when *skip != 0 the kernel returns at once (GMRES
// steps enqueued past a device-side stop).
void launch_reduce_partials(const double* partial, int nv, double* out, int take_sqrt,
                            cudaStream_t st, const int* skip = nullptr, int nparts = kRedBlocks);
// GMRES orthogonalisation passes (hbgpu_krylov.cu)
void launch_dcgs_dots(const double* V, long ld, int nv, const double* u, const double* w, long n,
                      double* partial, cudaStream_t st, const int* skip = nullptr);
void launch_dcgs_update(const double* V, long ld, int nv, const double* coef, double* u, double* w,
                        long n, double* partial, cudaStream_t st, const int* skip = nullptr);
// Short vectors (n <= kDots2dMax): 2-D grid dot pass over dcgs_dots_parts(n)
// element chunks (reduce with nparts = dcgs_dots_parts(n)).
constexpr long kDots2dMax = 1L << 20;
int dcgs_dots_parts(long n);
void launch_dcgs_dots2d(const double* V, long ld, int nv, const double* u, const double* w, long n,
                        double* partial, cudaStream_t st, const int* skip = nullptr);
int dcgs_update_parts(long n);
void launch_dcgs_update2(const double* V, long ld, int nv, const double* coef, double* u, double* w, long n,
                         double* partial, cudaStream_t st, const int* skip = nullptr);
// Device-resident Arnoldi/Givens state of one GMRES solve (hbgpu_krylov.cu).
struct ArnoldiDev {
    double* Hm;    // (m+2) x (m+1) Hessenberg, column-major, ld m+2
    double* R;     // its Givens-rotated copy
    double* cs;    // m+1
    double* sn;    // m+1
    double* gv;    // m+2
    double* hist;  // residual history indexed by iteration (hcap entries)
    int* ctl;      // [0] stop, [1] iterations, [2] final columns of the cycle, [3] reorthogonalisations
    int m, hcap;
};
// Step j of a cycle: from the reduced dot pass `red`, finalise column j-1
// (Givens, estimate, convergence test) and, unless the cycle ends, the
// tentative column j and the update coefficients.  d_norm = |w'_{j-1}|.
// H is row-major on the device, R column-major.
void launch_arnoldi_step(const ArnoldiDev& d, int j, int last, const double* red, const double* d_norm,
                         double* coef, double bnorm, double tol, cudaStream_t st);
size_t arnoldi_step_smem(int m);
cudaError_t configure_arnoldi_smem(int m);
// out = in/|in|, z = s*out, |in| = sqrt(sum of nparts partials) (also -> norm_out)
void launch_normalize_partials(const double* in, const double* partial, int nparts, double* norm_out,
                               double* out, const double* s, double* z, long n, cudaStream_t st,
                               const int* skip);
// Cycle start: zero H, R, gv; gv[0] = red0[0] = rnorm; ctl = {0, it, 0, reorth}.
void launch_arnoldi_init(const ArnoldiDev& d, double rnorm, int it, int reorth, double* red0,
                         cudaStream_t st);
void launch_basis_combine(const double* V, long ld, int nv, const double* y, const double* s,
                          double* x, long n, cudaStream_t st);
void launch_normalize(const double* in, const double* alpha, double* out, long n, cudaStream_t st,
                      const double* s = nullptr, double* z = nullptr, const int* skip = nullptr);

}  // namespace hbgpu
