// Krylov (GMRES) vector kernels — the orthogonalisation passes of
// gmres_solve (reference src/linalg.cpp:203-274).  HBM-bound: every pass
// streams the Krylov basis V once.  Reductions use a fixed partition of the
// vector into kRedBlocks contiguous chunks and fixed trees, so results are
// bit-reproducible run to run.
#include "hbgpu_internal.h"

#include <algorithm>
#include <cstdlib>

namespace hbgpu {

namespace {
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

__device__ __forceinline__ void chunk_of(long n, long& lo, long& hi) {
    const long chunk = (n + kRedBlocks - 1) / kRedBlocks;
    lo = (long)blockIdx.x * chunk;
    hi = lo + chunk < n ? lo + chunk : n;
}

// Block-wide sum of VB values per thread; results valid in threads 0..VB-1.
template <int VB>
__device__ __forceinline__ void block_sum_vec(double (&v)[VB], double (*red)[VB], double* out) {
#pragma unroll
    for (int q = 0; q < VB; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < VB; ++q)
            red[wid][q] = v[q];
    __syncthreads();
    if (threadIdx.x < VB) {
        double s = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k)
            s += red[k][threadIdx.x];
        out[threadIdx.x] = s;
    }
    __syncthreads();
}
}  // namespace

// Delayed-reorthogonalisation Arnoldi (DCGS2) dot pass: one read of
// V_0..V_{nv-1} gives a_i = <V_i, u> and b_i = <V_i, w>, plus <u,u>, <u,w>,
// <w,w>.  Row layout of `partial`: a (nv) | b (nv) | uu | uw | ww.  Without w
// (final step of a cycle): a (nv) | uu.
// The CTA's chunk is split into one contiguous segment per warp; all warps
// walk the same group of four basis vectors (so every warp has the same
// work), two elements per lane per iteration keep 12 loads in flight, and
// the per-warp sums are combined in warp order (fixed tree, deterministic).
__global__ void __launch_bounds__(kRedThreads) dcgs_dots_kernel(const double* __restrict__ V,
                                                                long ld, int nv,
                                                                const double* __restrict__ u,
                                                                const double* __restrict__ w,
                                                                long n, double* partial,
                                                                const int* skip) {
    if (skip && *skip)
        return;
    constexpr int NW = kRedThreads / 32;
    __shared__ double red[2][NW][8];
    long lo, hi;
    chunk_of(n, lo, hi);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long seg = (hi - lo + NW - 1) / NW;
    const long wlo = min(hi, lo + wid * seg), whi = min(hi, wlo + seg);
    const bool hw = w != nullptr;
    const int ngroups = (nv + 3) / 4;
    // groups 0..ngroups-1: basis vectors; group ngroups: the scalar products
    for (int g = 0; g <= ngroups; ++g) {
        const int buf = g & 1;
        double du[4] = {0.0, 0.0, 0.0, 0.0}, dw[4] = {0.0, 0.0, 0.0, 0.0};
        if (g < ngroups) {
            const int r0 = 4 * g, nr = min(4, nv - r0);
            const double* v0 = V + (long)r0 * ld;
            long k = wlo + lane;
            for (; k + 32 < whi; k += 64) {
                const double ua = u[k], ub = u[k + 32];
                const double wa = hw ? w[k] : 0.0, wb = hw ? w[k + 32] : 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q < nr) {
                        const double xa = __ldcs(v0 + (long)q * ld + k), xb = __ldcs(v0 + (long)q * ld + k + 32);
                        du[q] += xa * ua + xb * ub;
                        dw[q] += xa * wa + xb * wb;
                    }
            }
            for (; k < whi; k += 32) {
                const double ua = u[k], wa = hw ? w[k] : 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q < nr) {
                        const double xa = __ldcs(v0 + (long)q * ld + k);
                        du[q] += xa * ua;
                        dw[q] += xa * wa;
                    }
            }
        } else {
            for (long k = wlo + lane; k < whi; k += 32) {
                const double uk = u[k];
                du[0] += uk * uk;
                if (hw) {
                    const double wk = w[k];
                    du[1] += uk * wk;
                    du[2] += wk * wk;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                du[q] += __shfl_down_sync(0xffffffffu, du[q], o);
                dw[q] += __shfl_down_sync(0xffffffffu, dw[q], o);
            }
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                red[buf][wid][q] = du[q];
                red[buf][wid][4 + q] = dw[q];
            }
        __syncthreads();  // red[buf] complete; red[buf ^ 1] free for the next group
        if (threadIdx.x < 8) {
            const int c = threadIdx.x;
            double sum = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < NW; ++k2)
                sum += red[buf][k2][c];
            const int q = c & 3;
            if (g < ngroups) {
                const int r = 4 * g + q;
                if (r < nv) {
                    if (c < 4)
                        partial[(long)r * kRedBlocks + blockIdx.x] = sum;
                    else if (hw)
                        partial[(long)(nv + r) * kRedBlocks + blockIdx.x] = sum;
                }
            } else if (c < 3) {
                if (hw)
                    partial[(long)(2 * nv + c) * kRedBlocks + blockIdx.x] = sum;
                else if (c == 0)
                    partial[(long)nv * kRedBlocks + blockIdx.x] = sum;
            }
        }
    }
}

void launch_dcgs_dots(const double* V, long ld, int nv, const double* u, const double* w, long n,
                      double* partial, cudaStream_t st, const int* skip) {
    note_launch();
    dcgs_dots_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(V, ld, nv, u, w, n, partial, skip);
}

// The same dot pass for short vectors (n <= kDots2dMax): a 2-D grid, x = element
// chunk (nparts chunks of ~2048), y = group of eight basis vectors (the last
// group: <u,u>, <u,w>, <w,w>).  Every CTA issues all its loads up front and
// reduces once, so the pass is not a chain of per-group block reductions
// (config 0: 147,620-long vectors, ~40 us -> bandwidth-bound).  Same partial
// layout, nparts chunks per row.
constexpr int kDotsChunk = 2048;  // elements per chunk: 256 threads x 4 x double2
__global__ void __launch_bounds__(kRedThreads, 2) dcgs_dots2d_kernel(const double* __restrict__ V,
                                                                     long ld, int nv,
                                                                     const double* __restrict__ u,
                                                                     const double* __restrict__ w,
                                                                     long n, int nparts, double* partial,
                                                                     const int* skip) {
    if (skip && *skip)
        return;
    constexpr int NW = kRedThreads / 32, PER = kDotsChunk / (2 * kRedThreads);
    __shared__ double red[NW][16];
    const long lo = (long)blockIdx.x * kDotsChunk, hi = min(n, lo + kDotsChunk);
    const int g = blockIdx.y, ngroups = (nv + 7) / 8;
    const bool hw = w != nullptr;
    const bool full = hi - lo == kDotsChunk;  // rows are 16-byte aligned (n % 4 == 0)
    double du[8], dw[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
        du[q] = dw[q] = 0.0;
    if (g < ngroups) {
        const int r0 = 8 * g, nr = min(8, nv - r0);
        const double* v0 = V + (long)r0 * ld;
        if (full) {
            // every load of the chunk is independent: 4 x double2 per vector per thread
            double2 uu[PER], ww[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const long k = lo + 2L * (threadIdx.x + i * kRedThreads);
                uu[i] = *reinterpret_cast<const double2*>(u + k);
                ww[i] = hw ? *reinterpret_cast<const double2*>(w + k) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < nr) {
                    double2 x[PER];
#pragma unroll
                    for (int i = 0; i < PER; ++i)
                        x[i] = __ldcs(reinterpret_cast<const double2*>(v0 + (long)q * ld + lo +
                                                                       2L * (threadIdx.x + i * kRedThreads)));
#pragma unroll
                    for (int i = 0; i < PER; ++i) {
                        du[q] += x[i].x * uu[i].x + x[i].y * uu[i].y;
                        dw[q] += x[i].x * ww[i].x + x[i].y * ww[i].y;
                    }
                }
        } else {
            for (long k = lo + threadIdx.x; k < hi; k += blockDim.x) {
                const double uk = u[k], wk = hw ? w[k] : 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < nr) {
                        const double x = __ldcs(v0 + (long)q * ld + k);
                        du[q] += x * uk;
                        dw[q] += x * wk;
                    }
            }
        }
    } else {
        for (long k = lo + threadIdx.x; k < hi; k += blockDim.x) {
            const double uk = u[k];
            du[0] += uk * uk;
            if (hw) {
                const double wk = w[k];
                du[1] += uk * wk;
                du[2] += wk * wk;
            }
        }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            du[q] += __shfl_down_sync(0xffffffffu, du[q], o);
            dw[q] += __shfl_down_sync(0xffffffffu, dw[q], o);
        }
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            red[wid][q] = du[q];
            red[wid][8 + q] = dw[q];
        }
    __syncthreads();
    if (threadIdx.x < 16) {
        const int c = threadIdx.x, q = c & 7;
        double sum = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < NW; ++k2)
            sum += red[k2][c];
        if (g < ngroups) {
            const int r = 8 * g + q;
            if (r < nv) {
                if (c < 8)
                    partial[(long)r * kRedBlocks + blockIdx.x] = sum;
                else if (hw)
                    partial[(long)(nv + r) * kRedBlocks + blockIdx.x] = sum;
            }
        } else if (c < 3) {
            if (hw)
                partial[(long)(2 * nv + c) * kRedBlocks + blockIdx.x] = sum;
            else if (c == 0)
                partial[(long)nv * kRedBlocks + blockIdx.x] = sum;
        }
    }
}

int dcgs_dots_parts(long n) {
    if (n > kDots2dMax)
        return kRedBlocks;
    const long p = (n + kDotsChunk - 1) / kDotsChunk;
    return (int)(p < 1 ? 1 : (p > kRedBlocks ? kRedBlocks : p));
}

void launch_dcgs_dots2d(const double* V, long ld, int nv, const double* u, const double* w, long n,
                        double* partial, cudaStream_t st, const int* skip) {
    note_launch();
    const dim3 grid(dcgs_dots_parts(n), (nv + 7) / 8 + 1);
    dcgs_dots2d_kernel<<<grid, kRedThreads, 0, st>>>(V, ld, nv, u, w, n, (int)grid.x, partial, skip);
}

// DCGS2 update pass, one read of V_0..V_{nv-1}:
//   q  = (u - sum_i a_i V_i) / rho                  (re-orthogonalised previous vector, in place of u)
//   w' = (w - cr u - sum_i d_i V_i) / rho           (projected new vector, in place of w)
// and the block partial of ||w'||^2.  coef = [a (nv) | d (nv) | 1/rho | cr].
__global__ void __launch_bounds__(kRedThreads) dcgs_update_kernel(const double* __restrict__ V,
                                                                  long ld, int nv,
                                                                  const double* __restrict__ coef,
                                                                  double* __restrict__ u,
                                                                  double* __restrict__ w, long n,
                                                                  double* partial, const int* skip) {
    if (skip && *skip)
        return;
    extern __shared__ double cs[];
    for (int i = threadIdx.x; i < 2 * nv + 2; i += blockDim.x)
        cs[i] = coef[i];
    __syncthreads();
    __shared__ double red[kRedThreads / 32][1];
    __shared__ double res[1];
    const double* ca = cs;
    const double* cd = cs + nv;
    const double inv_rho = cs[2 * nv], cr = cs[2 * nv + 1];
    double acc[1] = {0.0};
    for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (long)gridDim.x * blockDim.x) {
        double sa0 = 0.0, sa1 = 0.0, sd0 = 0.0, sd1 = 0.0;
        int i = 0;
        for (; i + 7 < nv; i += 8) {  // eight basis vectors in flight per thread
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                v[q] = __ldcs(V + (long)(i + q) * ld + k);
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
                sa0 += ca[i + q] * v[q];
                sa1 += ca[i + q + 1] * v[q + 1];
                sd0 += cd[i + q] * v[q];
                sd1 += cd[i + q + 1] * v[q + 1];
            }
        }
        for (; i + 3 < nv; i += 4) {
            const double v0 = __ldcs(V + (long)i * ld + k), v1 = __ldcs(V + (long)(i + 1) * ld + k);
            const double v2 = __ldcs(V + (long)(i + 2) * ld + k), v3 = __ldcs(V + (long)(i + 3) * ld + k);
            sa0 += ca[i] * v0;
            sa1 += ca[i + 1] * v1;
            sd0 += cd[i] * v0;
            sd1 += cd[i + 1] * v1;
            sa0 += ca[i + 2] * v2;
            sa1 += ca[i + 3] * v3;
            sd0 += cd[i + 2] * v2;
            sd1 += cd[i + 3] * v3;
        }
        for (; i + 1 < nv; i += 2) {
            const double v0 = __ldcs(V + (long)i * ld + k), v1 = __ldcs(V + (long)(i + 1) * ld + k);
            sa0 += ca[i] * v0;
            sa1 += ca[i + 1] * v1;
            sd0 += cd[i] * v0;
            sd1 += cd[i + 1] * v1;
        }
        if (i < nv) {
            const double v0 = __ldcs(V + (long)i * ld + k);
            sa0 += ca[i] * v0;
            sd0 += cd[i] * v0;
        }
        const double uk = u[k];
        u[k] = (uk - (sa0 + sa1)) * inv_rho;
        const double wn = (w[k] - cr * uk - (sd0 + sd1)) * inv_rho;
        w[k] = wn;
        acc[0] += wn * wn;
    }
    block_sum_vec<1>(acc, red, res);
    if (threadIdx.x == 0)
        partial[blockIdx.x] = res[0];
}

void launch_dcgs_update(const double* V, long ld, int nv, const double* coef, double* u, double* w,
                        long n, double* partial, cudaStream_t st, const int* skip) {
    note_launch();
    dcgs_update_kernel<<<kRedBlocks, kRedThreads, sizeof(double) * (2 * nv + 2), st>>>(
        V, ld, nv, coef, u, w, n, partial, skip);
}

// The update pass of the device-resident cycle (n % 4 == 0): thread per pair
// of elements (16-byte loads), sixteen basis vectors in flight, grid of
// dcgs_update_parts(n) CTAs (one ||w'||^2 partial each).  Config 1 (n = 4.06M,
// 100 basis vectors): 670 -> 553 us (6.1 TB/s) against dcgs_update_kernel.
__global__ void __launch_bounds__(kRedThreads) dcgs_update2_kernel(const double* __restrict__ V,
                                                                   long ld, int nv,
                                                                   const double* __restrict__ coef,
                                                                   double* __restrict__ u,
                                                                   double* __restrict__ w, long n,
                                                                   double* partial, const int* skip) {
    if (skip && *skip)
        return;
    extern __shared__ double cs[];
    for (int i = threadIdx.x; i < 2 * nv + 2; i += blockDim.x)
        cs[i] = coef[i];
    __syncthreads();
    __shared__ double red[kRedThreads / 32][1];
    __shared__ double res[1];
    const double* ca = cs;
    const double* cd = cs + nv;
    const double inv_rho = cs[2 * nv], cr = cs[2 * nv + 1];
    double acc[1] = {0.0};
    for (long k = 2 * ((long)blockIdx.x * blockDim.x + threadIdx.x); k < n; k += 2L * gridDim.x * blockDim.x) {
        double2 sa = make_double2(0.0, 0.0), sd = make_double2(0.0, 0.0);
        for (int i = 0; i < nv; i += 16) {
            double2 v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
                v[q] = (i + q < nv) ? __ldcs(reinterpret_cast<const double2*>(V + (long)(i + q) * ld + k))
                                    : make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 16; ++q)
                if (i + q < nv) {
                    const double a = ca[i + q], dd = cd[i + q];
                    sa.x += a * v[q].x;
                    sa.y += a * v[q].y;
                    sd.x += dd * v[q].x;
                    sd.y += dd * v[q].y;
                }
        }
        const double2 uk = *reinterpret_cast<const double2*>(u + k);
        const double2 wk = *reinterpret_cast<const double2*>(w + k);
        *reinterpret_cast<double2*>(u + k) = make_double2((uk.x - sa.x) * inv_rho, (uk.y - sa.y) * inv_rho);
        const double2 wn = make_double2((wk.x - cr * uk.x - sd.x) * inv_rho, (wk.y - cr * uk.y - sd.y) * inv_rho);
        *reinterpret_cast<double2*>(w + k) = wn;
        acc[0] += wn.x * wn.x + wn.y * wn.y;
    }
    block_sum_vec<1>(acc, red, res);
    if (threadIdx.x == 0)
        partial[blockIdx.x] = res[0];
}

int dcgs_update_parts(long n) {
    if (n > kDots2dMax)
        return kRedBlocks;
    const long per = 2L * kRedThreads;
    const long p = (n + per - 1) / per;
    return (int)(p < 1 ? 1 : (p > kRedBlocks ? kRedBlocks : p));
}

void launch_dcgs_update2(const double* V, long ld, int nv, const double* coef, double* u, double* w, long n,
                         double* partial, cudaStream_t st, const int* skip) {
    note_launch();
    dcgs_update2_kernel<<<dcgs_update_parts(n), kRedThreads, sizeof(double) * (2 * nv + 2), st>>>(
        V, ld, nv, coef, u, w, n, partial, skip);
}

// x <- x + s * sum_i y_i V_i (solution update x += S V y, linalg.cpp:272-274).
__global__ void __launch_bounds__(kRedThreads) basis_combine_kernel(const double* __restrict__ V,
                                                                    long ld, int nv,
                                                                    const double* __restrict__ y,
                                                                    const double* __restrict__ s,
                                                                    double* __restrict__ x, long n) {
    extern __shared__ double ys[];
    for (int i = threadIdx.x; i < nv; i += blockDim.x)
        ys[i] = y[i];
    __syncthreads();
    for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (long)gridDim.x * blockDim.x) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int i = 0;
        for (; i + 3 < nv; i += 4) {
            s0 += ys[i] * __ldcs(V + (long)i * ld + k);
            s1 += ys[i + 1] * __ldcs(V + (long)(i + 1) * ld + k);
            s2 += ys[i + 2] * __ldcs(V + (long)(i + 2) * ld + k);
            s3 += ys[i + 3] * __ldcs(V + (long)(i + 3) * ld + k);
        }
        for (; i < nv; ++i)
            s0 += ys[i] * __ldcs(V + (long)i * ld + k);
        x[k] += s[k] * ((s0 + s1) + (s2 + s3));
    }
}

void launch_basis_combine(const double* V, long ld, int nv, const double* y, const double* s,
                          double* x, long n, cudaStream_t st) {
    note_launch();
    basis_combine_kernel<<<8 * 148, kRedThreads, sizeof(double) * (nv > 0 ? nv : 1), st>>>(
        V, ld, nv, y, s, x, n);
}

// out = in / alpha[0] (alpha on device; zero when alpha == 0, breakdown) and,
// when s is given, z = s * out — the scaled input of the next S A S product
// (linalg.cpp:214-216), produced in the same pass.
__global__ void normalize_kernel(const double* __restrict__ in, const double* __restrict__ alpha,
                                 double* __restrict__ out, const double* __restrict__ s,
                                 double* __restrict__ z, long n, const int* skip) {
    if (skip && *skip)
        return;
    const double a = *alpha;
    for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (long)gridDim.x * blockDim.x) {
        const double v = a != 0.0 ? in[k] / a : 0.0;
        out[k] = v;
        if (s)
            z[k] = s[k] * v;
    }
}

void launch_normalize(const double* in, const double* alpha, double* out, long n,
                      cudaStream_t st, const double* s, double* z, const int* skip) {
    note_launch();
    normalize_kernel<<<8 * 148, 256, 0, st>>>(in, alpha, out, s, z, n, skip);
}

// ---------------------------------------------------------------- Arnoldi step
// The small dense part of one DCGS2 GMRES step (what gmres_dev's host loop
// does between the dot pass and the update pass, see hbgpu_host.cu), so a
// cycle runs without a host round trip per step:
//   rho = sqrt(<u,u> - |a|^2) from the reduced dot pass;
//   column j-1 is finalised with the re-orthogonalisation of u_j, rotated
//   (Givens, linalg.cpp:237-258), and the residual estimate / convergence /
//   breakdown test sets ctl[0];  unless the cycle ends, the tentative column
//   j = (c - H_j a)/rho and the update coefficients [a | b - cr a | 1/rho | cr].
// One CTA of 256.  H is row-major (row i contiguous), so the O(j^2) product
// H_j a is read as (row, 32-column segment) items, each a run of independent
// loads; warp 0 runs the Givens chain on shared-memory copies meanwhile.
// Every sum has a fixed order (deterministic).
constexpr int kArnThreads = 256;
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_down_sync(0xffffffffu, v, o);
    return v;  // lane 0
}

__device__ __forceinline__ void arnoldi_step_body(const ArnoldiDev& d, int j, int last,
                                                  const double* __restrict__ red,
                                                  const double* __restrict__ d_norm,
                                                  double* __restrict__ coef, double bnorm, double tol,
                                                  double* __restrict__ sh) {
    if (*(volatile int*)d.ctl)
        return;
    const int m = d.m, ldh = m + 1;    // H row-major: H(i, l) = Hm[i * ldh + l]
    const size_t ldr = (size_t)m + 2;  // R column-major
    double* av = sh;                   // j
    double* bv = av + (m + 1);         // j
    double* gcs = bv + (m + 1);        // Givens copies: cs, sn (k), column k (k + 2)
    double* gsn = gcs + (m + 1);
    double* grc = gsn + (m + 1);
    double* hkc = grc + (m + 2);       // finalised column k, unrotated
    double* ps = hkc + (m + 2);        // (j + 1) x nseg partial row products
    __shared__ double s_sc[6];         // uu, uw, aa, ab, |w'_{j-1}|, gv[k]
    __shared__ double s_rho, s_cj;
    __shared__ int s_stop;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = j - 1;
    const bool tent = !last;  // the tentative column j is needed (unless rho = 0 or stop)
    // A. every independent global read at once: dot results, column k of H,
    //    the Givens history, |w'_{j-1}|, gv[k]
    for (int i = tid; i < j; i += kArnThreads) {
        av[i] = red[i];
        if (!last)
            bv[i] = red[j + i];
        grc[i] = d.Hm[(size_t)i * ldh + k];
        if (i < k) {
            gcs[i] = d.cs[i];
            gsn[i] = d.sn[i];
        }
    }
    if (tid == 0) {
        s_sc[0] = last ? red[j] : red[2 * j];
        s_sc[1] = last ? 0.0 : red[2 * j + 1];
        s_sc[4] = j >= 1 ? *d_norm : 0.0;
        s_sc[5] = j >= 1 ? d.gv[k] : 0.0;
        s_stop = 0;
    }
    __syncthreads();
    // B. |a|^2 (warp 0), a.b (warp 1); warps 2.. the part of H_j a over the
    //    final columns l < k (row i, 32-column segment items)
    const int nseg = (j + 31) / 32;
    if (warp < 2) {
        if (warp == 0 || !last) {
            double acc = 0.0;
            for (int i = lane; i < j; i += 32)
                acc += av[i] * (warp == 0 ? av[i] : bv[i]);
            acc = warp_sum(acc);
            if (lane == 0)
                s_sc[2 + warp] = acc;
        }
    } else if (tent) {
        for (int it = tid - 64; it < (j + 1) * nseg; it += kArnThreads - 64) {
            const int i = it / nseg, sg = it - i * nseg;
            const int l0 = max(32 * sg, i - 1), l1 = min(k, 32 * sg + 32);
            const double* hr = d.Hm + (size_t)i * ldh;
            double acc = 0.0;
            if (l0 < l1) {
                double v[32];
#pragma unroll
                for (int q = 0; q < 32; ++q)
                    v[q] = (l0 + q < l1) ? hr[l0 + q] : 0.0;
#pragma unroll
                for (int q = 0; q < 32; ++q)
                    if (l0 + q < l1)
                        acc += v[q] * av[l0 + q];
            }
            ps[it] = acc;
        }
    }
    __syncthreads();
    if (tid == 0) {
        const double rho2 = s_sc[0] - s_sc[2];
        const double rho = rho2 > 0.0 ? sqrt(rho2) : 0.0;
        s_rho = rho;
        s_cj = (!last && rho > 0.0) ? (s_sc[1] - s_sc[3]) / rho : 0.0;
    }
    __syncthreads();
    const double rho = s_rho;
    // C. finalise column k = j-1 with the re-orthogonalisation of u_j:
    //    H[0:j, k] += |w'_{j-1}| a,  H[j, k] = |w'_{j-1}| rho
    if (j >= 1) {
        const double hjj1 = s_sc[4];
        for (int i = tid; i <= j; i += kArnThreads) {
            const double h = i < j ? grc[i] + hjj1 * av[i] : hjj1 * rho;
            grc[i] = h;
            hkc[i] = h;
            d.Hm[(size_t)i * ldh + k] = h;
        }
    }
    __syncthreads();
    if (warp == 0) {
        if (j >= 1 && lane == 0) {
            // D. Givens rotations of column k (chain in registers, operands in smem)
            const bool zero_sub = grc[j] == 0.0;
            double x = grc[0];
#pragma unroll 4
            for (int i = 0; i < k; ++i) {
                const double y = grc[i + 1], c = gcs[i], sg = gsn[i];
                grc[i] = c * x + sg * y;
                x = -sg * x + c * y;
            }
            const double xk1 = grc[k + 1];
            const double den = hypot(x, xk1);
            const double c = den == 0.0 ? 1.0 : x / den;
            const double sg = den == 0.0 ? 0.0 : xk1 / den;
            d.cs[k] = c;
            d.sn[k] = sg;
            grc[k] = den;
            grc[k + 1] = 0.0;
            const double gk = s_sc[5];
            d.gv[k + 1] = -sg * gk;
            d.gv[k] = c * gk;
            const int it = d.ctl[1] + 1;
            d.ctl[1] = it;
            d.ctl[2] = j;
            d.ctl[3] += 1;
            const double est = fabs(sg * gk);
            if (it < d.hcap)
                d.hist[it] = est / bnorm;
            if (est / bnorm <= tol || zero_sub)
                s_stop = 1;
        }
    } else if (tent && rho > 0.0) {
        // D'. tentative column j: h_i = ((i < j ? b_i : cj) - H_j a) / rho, with
        //     the finalised column k added to the partial products
        const double cj = s_cj, ak = j >= 1 ? av[k] : 0.0;
        for (int i = tid - 32; i <= j; i += kArnThreads - 32) {
            double ha = 0.0;
            for (int sg = 0; sg < nseg; ++sg)
                ha += ps[i * nseg + sg];
            if (j >= 1)
                ha += hkc[i] * ak;
            d.Hm[(size_t)i * ldh + j] = ((i < j ? bv[i] : cj) - ha) / rho;
        }
    }
    __syncthreads();
    if (j >= 1)
        for (int i = tid; i <= j; i += kArnThreads)
            d.R[(size_t)k * ldr + i] = grc[i];
    if (last)
        return;
    if (s_stop || !(rho > 0.0)) {  // converged, or u_j in span(Q) (breakdown)
        if (tid == 0)
            d.ctl[0] = 1;
        return;
    }
    const double cr = s_cj / rho;
    for (int i = tid; i < j; i += kArnThreads) {
        coef[i] = av[i];
        coef[j + i] = bv[i] - cr * av[i];
    }
    if (tid == 0) {
        coef[2 * j] = 1.0 / rho;
        coef[2 * j + 1] = cr;
        if (j == 0)
            d.gv[0] *= rho;  // V_0 renormalised by its computed norm in the update pass
    }
}

__global__ void __launch_bounds__(kArnThreads) arnoldi_step_kernel(ArnoldiDev d, int j, int last,
                                                                   const double* __restrict__ red,
                                                                   const double* __restrict__ d_norm,
                                                                   double* __restrict__ coef, double bnorm,
                                                                   double tol) {
    extern __shared__ double sh[];
    arnoldi_step_body(d, j, last, red, d_norm, coef, bnorm, tol, sh);
}

void launch_arnoldi_step(const ArnoldiDev& d, int j, int last, const double* red, const double* d_norm,
                         double* coef, double bnorm, double tol, cudaStream_t st) {
    note_launch();
    const int nseg = (j + 31) / 32;
    const size_t smem = sizeof(double) * (6 * (size_t)d.m + 8 + (size_t)(j + 1) * (nseg > 0 ? nseg : 1));
    arnoldi_step_kernel<<<1, kArnThreads, smem, st>>>(d, j, last, red, d_norm, coef, bnorm, tol);
}

size_t arnoldi_step_smem(int m) {
    return sizeof(double) * (6 * (size_t)m + 8 + (size_t)(m + 1) * (size_t)((m + 31) / 32));
}

cudaError_t configure_arnoldi_smem(int m) {
    return cudaFuncSetAttribute(arnoldi_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)arnoldi_step_smem(m));
}

// V_{j+1} = w' / |w'| and z = s V_{j+1}, with |w'| = sqrt of the update pass's
// nparts partials summed in fixed order by every CTA (CTA 0 stores it for the
// next Arnoldi step): one launch instead of reduce + normalize.
__global__ void normalize_partials_kernel(const double* __restrict__ in,
                                          const double* __restrict__ partial, int nparts,
                                          double* __restrict__ norm_out, double* __restrict__ out,
                                          const double* __restrict__ s, double* __restrict__ z, long n,
                                          const int* skip) {
    if (skip && *skip)
        return;
    __shared__ double red[8];
    __shared__ double s_a;
    double acc = 0.0;
    for (int q = threadIdx.x; q < nparts; q += blockDim.x)
        acc += partial[q];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            t += red[w];
        s_a = sqrt(t);
        if (blockIdx.x == 0)
            *norm_out = s_a;
    }
    __syncthreads();
    const double a = s_a;
    for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
        const double v = a != 0.0 ? in[k] / a : 0.0;
        out[k] = v;
        z[k] = s[k] * v;
    }
}

void launch_normalize_partials(const double* in, const double* partial, int nparts, double* norm_out,
                               double* out, const double* s, double* z, long n, cudaStream_t st,
                               const int* skip) {
    note_launch();
    const long per = 256L * 4;
    const int blocks = (int)std::min<long>(8 * 148, (n + per - 1) / per);
    normalize_partials_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(in, partial, nparts, norm_out, out, s, z,
                                                                       n, skip);
}

__global__ void arnoldi_init_kernel(ArnoldiDev d, double rnorm, int it, int reorth, double* red0) {
    const size_t nhr = ((size_t)d.m + 2) * ((size_t)d.m + 1);
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < nhr; k += (size_t)gridDim.x * blockDim.x) {
        d.Hm[k] = 0.0;
        d.R[k] = 0.0;
        if (k < (size_t)d.m + 2)
            d.gv[k] = k == 0 ? rnorm : 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        d.ctl[0] = 0;
        d.ctl[1] = it;
        d.ctl[2] = 0;
        d.ctl[3] = reorth;
        red0[0] = rnorm;
    }
}

void launch_arnoldi_init(const ArnoldiDev& d, double rnorm, int it, int reorth, double* red0,
                         cudaStream_t st) {
    note_launch();
    arnoldi_init_kernel<<<64, 256, 0, st>>>(d, rnorm, it, reorth, red0);
}

}  // namespace hbgpu
