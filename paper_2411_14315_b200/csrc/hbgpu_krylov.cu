// Krylov (GMRES) vector kernels — the orthogonalisation passes of
// gmres_solve (reference src/linalg.cpp:203-274).  HBM-bound: every pass
// streams the Krylov basis V once.  Reductions use a fixed partition of the
// vector into kRedBlocks contiguous chunks and fixed trees, so results are
// bit-reproducible run to run.
#include "hbgpu_internal.h"

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
__global__ void __launch_bounds__(kRedThreads) dcgs_dots_kernel(const double* __restrict__ V,
                                                                long ld, int nv,
                                                                const double* __restrict__ u,
                                                                const double* __restrict__ w,
                                                                long n, double* partial) {
    long lo, hi;
    chunk_of(n, lo, hi);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool hw = w != nullptr;
    // tasks: groups of four basis vectors (u and w read once per group), then
    // the three scalar products
    const int ngroups = (nv + 3) / 4;
    for (int task = wid; task < ngroups; task += nw) {
        const int r0 = 4 * task, nr = min(4, nv - r0);
        double du[4] = {0.0, 0.0, 0.0, 0.0}, dw[4] = {0.0, 0.0, 0.0, 0.0};
        for (long k = lo + lane; k < hi; k += 32) {
            const double uk = u[k];
            const double wk = hw ? w[k] : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (q < nr) {
                    const double x = V[(long)(r0 + q) * ld + k];
                    du[q] += x * uk;
                    dw[q] += x * wk;
                }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                du[q] += __shfl_down_sync(0xffffffffu, du[q], o);
                dw[q] += __shfl_down_sync(0xffffffffu, dw[q], o);
            }
            if (lane == 0 && q < nr) {
                partial[(long)(r0 + q) * kRedBlocks + blockIdx.x] = du[q];
                if (hw)
                    partial[(long)(nv + r0 + q) * kRedBlocks + blockIdx.x] = dw[q];
            }
        }
    }
    if (wid == (ngroups % nw)) {  // the scalar task goes to the least loaded warp
        const int r = nv;
        double du0 = 0.0, du1 = 0.0, dw0 = 0.0, dw1 = 0.0, dx0 = 0.0, dx1 = 0.0;
        if (r < nv) {
            const double* x = V + (long)r * ld;
            long k = lo + lane;
            for (; k + 32 < hi; k += 64) {
                const double x0 = x[k], x1 = x[k + 32];
                du0 += x0 * u[k];
                du1 += x1 * u[k + 32];
                if (hw) {
                    dw0 += x0 * w[k];
                    dw1 += x1 * w[k + 32];
                }
            }
            for (; k < hi; k += 32) {
                du0 += x[k] * u[k];
                if (hw)
                    dw0 += x[k] * w[k];
            }
        } else {
            long k = lo + lane;
            for (; k < hi; k += 32) {
                const double uk = u[k];
                du0 += uk * uk;
                if (hw) {
                    const double wk = w[k];
                    dw0 += uk * wk;
                    dx0 += wk * wk;
                }
            }
        }
        double su = du0 + du1, sw = dw0 + dw1, sx = dx0 + dx1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            su += __shfl_down_sync(0xffffffffu, su, o);
            sw += __shfl_down_sync(0xffffffffu, sw, o);
            sx += __shfl_down_sync(0xffffffffu, sx, o);
        }
        if (lane == 0) {
            if (r < nv) {
                partial[(long)r * kRedBlocks + blockIdx.x] = su;
                if (hw)
                    partial[(long)(nv + r) * kRedBlocks + blockIdx.x] = sw;
            } else if (hw) {
                partial[(long)(2 * nv) * kRedBlocks + blockIdx.x] = su;
                partial[(long)(2 * nv + 1) * kRedBlocks + blockIdx.x] = sw;
                partial[(long)(2 * nv + 2) * kRedBlocks + blockIdx.x] = sx;
            } else {
                partial[(long)nv * kRedBlocks + blockIdx.x] = su;
            }
        }
    }
}

void launch_dcgs_dots(const double* V, long ld, int nv, const double* u, const double* w, long n,
                      double* partial, cudaStream_t st) {
    note_launch();
    dcgs_dots_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(V, ld, nv, u, w, n, partial);
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
                                                                  double* partial) {
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
                        long n, double* partial, cudaStream_t st) {
    note_launch();
    dcgs_update_kernel<<<kRedBlocks, kRedThreads, sizeof(double) * (2 * nv + 2), st>>>(
        V, ld, nv, coef, u, w, n, partial);
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
                                 double* __restrict__ z, long n) {
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
                      cudaStream_t st, const double* s, double* z) {
    note_launch();
    normalize_kernel<<<8 * 148, 256, 0, st>>>(in, alpha, out, s, z, n);
}

}  // namespace hbgpu
