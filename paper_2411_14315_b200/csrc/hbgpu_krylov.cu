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
// The CTA's chunk is split into one contiguous segment per warp; all warps
// walk the same group of four basis vectors (so every warp has the same
// work), two elements per lane per iteration keep 12 loads in flight, and
// the per-warp sums are combined in warp order (fixed tree, deterministic).
__global__ void __launch_bounds__(kRedThreads) dcgs_dots_kernel(const double* __restrict__ V,
                                                                long ld, int nv,
                                                                const double* __restrict__ u,
                                                                const double* __restrict__ w,
                                                                long n, double* partial) {
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
