// Fused L-matvec (TangentOperator::matvec, reference src/linalg.cpp:78-128):
//   out_A = sum_k P_k y_col(k) + [A free] H * sum_{k: col free} m_k y_col(k)[velocity]
// HBM-bound: P.vals (64 N bytes per block) dominates the traffic and is
// streamed exactly once with evict-first loads; y stays L2/L1 resident.
#include "hbgpu_internal.h"

namespace hbgpu {

namespace {
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

__device__ __forceinline__ double ldcs(const double* p) {
#if MV_PREFETCH == 1
    double v;
    asm volatile("ld.global.cs.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#elif MV_PREFETCH == 2
    double v;
    asm volatile("ld.global.L1::no_allocate.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#elif MV_PREFETCH == 3
    double v;
    asm volatile("ld.global.cs.L2::128B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}
__device__ __forceinline__ double2 ldcs2(const double2* p) { return __ldcs(p); }
}  // namespace

// Thread (row, n).  The Dirichlet masks of C are folded into `mass_c`
// (m_k = 0 when row or column is constrained, linalg.cpp:109,115), so the
// block loop is branch-free; two blocks per iteration keep 24+ independent
// loads in flight per thread.  The N threads of a row exchange the gathered
// velocity series through shared memory for the dense H product.
// N1: N == 1 (steady / time-stepping case): a block's 8 slots are 64 contiguous
// bytes and y's 4 components 32 — loaded as 16-byte vectors (H is 0, no C part).
#ifndef MV_CTA_THREADS
#define MV_CTA_THREADS 512
#endif
#ifndef MV_UNROLL4
#define MV_UNROLL4 0
#endif
template <bool SCALED, bool WITH_C, bool N1>
__global__ void __launch_bounds__(MV_CTA_THREADS) lmatvec_kernel(MatvecArgs a) {
    if (a.skip && *a.skip)
        return;
    extern __shared__ double sh[];
    const int N = a.N;
    double* sH = sh;
    double* st = sh + (WITH_C ? N * N : 0);
    if (WITH_C)
        for (int k = threadIdx.x; k < N * N; k += blockDim.x)
            sH[k] = a.H[k];
    const int r = threadIdx.x / N, n = threadIdx.x - r * N;
    const int ridx = blockIdx.x * a.rows_per_cta + r;
    const bool valid = (r < a.rows_per_cta) && (ridx < a.nn);
    int A = ridx, kb = 0, ke = 0;
    if (valid) {
        if (a.rows) {  // {A, row_ptr[A], row_ptr[A+1]} in one load
            const int4 rr = __ldg(a.rows + ridx);
            A = rr.x;
            kb = rr.y;
            ke = rr.z;
        } else {
            A = a.perm ? __ldg(a.perm + ridx) : ridx;
            kb = a.row_ptr[A];
            ke = a.row_ptr[A + 1];
        }
    }
    double ou0 = 0.0, ou1 = 0.0, ou2 = 0.0, op = 0.0, t0 = 0.0, t1 = 0.0, t2 = 0.0;
    const long N8 = 8L * N;
    auto block = [&](int k, int B) {
        double y0, y1, y2, y3, kd, g0, g1, g2, d0, d1, d2, ld;
        if (N1) {
            const double2* v = reinterpret_cast<const double2*>(a.vals + (long)k * 8);
            const double2* yv = reinterpret_cast<const double2*>(a.y + (long)B * 4);
            const double2 ya = __ldg(yv), yb2 = __ldg(yv + 1);
            const double2 p0 = __ldcs(v), p1 = __ldcs(v + 1), p2 = __ldcs(v + 2), p3 = __ldcs(v + 3);
            y0 = ya.x; y1 = ya.y; y2 = yb2.x; y3 = yb2.y;
            kd = p0.x; g0 = p0.y; g1 = p1.x; g2 = p1.y; d0 = p2.x; d1 = p2.y; d2 = p3.x; ld = p3.y;
        } else {
            const double* v = a.vals + (long)k * N8 + n;
            const long yb = (long)B * 4 * N + n;
            y0 = __ldg(a.y + yb);
            y1 = __ldg(a.y + yb + N);
            y2 = __ldg(a.y + yb + 2 * N);
            y3 = __ldg(a.y + yb + 3 * N);
            kd = ldcs(v);
            g0 = ldcs(v + N);
            g1 = ldcs(v + 2 * N);
            g2 = ldcs(v + 3 * N);
            d0 = ldcs(v + 4 * N);
            d1 = ldcs(v + 5 * N);
            d2 = ldcs(v + 6 * N);
            ld = ldcs(v + 7 * N);
        }
        ou0 += kd * y0 + g0 * y3;
        ou1 += kd * y1 + g1 * y3;
        ou2 += kd * y2 + g2 * y3;
        op += d0 * y0;
        op += d1 * y1;
        op += d2 * y2;
        op += ld * y3;
        if (WITH_C) {
            const double m = __ldg(a.mass + k);
            t0 += m * y0;
            t1 += m * y1;
            t2 += m * y2;
        }
    };
    if (valid) {
        int k = kb;
        // (loading the next blocks' column indices one iteration ahead measured
        // 25% slower on every mesh: more registers, fewer loads in flight)
        {
#if MV_UNROLL4
            for (; k + 3 < ke; k += 4) {
                const int B0 = __ldg(a.col_idx + k), B1 = __ldg(a.col_idx + k + 1);
                const int B2 = __ldg(a.col_idx + k + 2), B3 = __ldg(a.col_idx + k + 3);
                block(k, B0);
                block(k + 1, B1);
                block(k + 2, B2);
                block(k + 3, B3);
            }
#endif
            for (; k + 1 < ke; k += 2) {
                block(k, __ldg(a.col_idx + k));
                block(k + 1, __ldg(a.col_idx + k + 1));
            }
            if (k < ke)
                block(k, __ldg(a.col_idx + k));
        }
    }
    if (WITH_C) {
        if (valid) {
            st[(r * 3 + 0) * N + n] = t0;
            st[(r * 3 + 1) * N + n] = t1;
            st[(r * 3 + 2) * N + n] = t2;
        }
        __syncthreads();
        if (valid) {
            const double* h = sH + n * N;
            const double* s0 = st + (r * 3) * N;
            double h0 = 0.0, h1 = 0.0, h2 = 0.0;
            for (int m = 0; m < N; ++m) {
                const double hm = h[m];
                h0 += hm * s0[m];
                h1 += hm * s0[N + m];
                h2 += hm * s0[2 * N + m];
            }
            ou0 += h0;
            ou1 += h1;
            ou2 += h2;
        }
    }
    if (valid) {
        const long o = (long)A * 4 * N + n;
        if (SCALED) {
            ou0 *= __ldg(a.scale_out + o);
            ou1 *= __ldg(a.scale_out + o + N);
            ou2 *= __ldg(a.scale_out + o + 2 * N);
            op *= __ldg(a.scale_out + o + 3 * N);
        }
        a.out[o] = ou0;
        a.out[o + N] = ou1;
        a.out[o + 2 * N] = ou2;
        a.out[o + 3 * N] = op;
    }
}

static void launch_main(const MatvecArgs& a, int blocks, int threads, size_t smem, cudaStream_t st) {
    if (a.N == 1) {  // H = 0: P only
        if (a.scale_out)
            lmatvec_kernel<true, false, true><<<blocks, threads, 0, st>>>(a);
        else
            lmatvec_kernel<false, false, true><<<blocks, threads, 0, st>>>(a);
    } else if (a.with_c) {
        if (a.scale_out)
            lmatvec_kernel<true, true, false><<<blocks, threads, smem, st>>>(a);
        else
            lmatvec_kernel<false, true, false><<<blocks, threads, smem, st>>>(a);
    } else {
        if (a.scale_out)
            lmatvec_kernel<true, false, false><<<blocks, threads, smem, st>>>(a);
        else
            lmatvec_kernel<false, false, false><<<blocks, threads, smem, st>>>(a);
    }
}

// N > 1 with G lanes per (row, sample): thread (r, g, n) takes the row's
// blocks kb+g, kb+g+G, ...; the G partial sums are combined in g order
// through shared memory (deterministic).  Shorter per-thread block chains for
// meshes too small to fill the GPU with (row, sample) threads alone.
template <bool SCALED, bool WITH_C, int G>
__global__ void __launch_bounds__(256) lmatvec_g_kernel(MatvecArgs a) {
    if (a.skip && *a.skip)
        return;
    extern __shared__ double sh[];
    const int N = a.N, rpc = a.rows_per_cta;
    double* sH = sh;
    double* st = sh + (WITH_C ? N * N : 0);
    double* pr = st + (WITH_C ? 3 * N * rpc : 0);  // [r][g][7][N]
    if (WITH_C)
        for (int k = threadIdx.x; k < N * N; k += blockDim.x)
            sH[k] = a.H[k];
    const int GN = G * N;
    const int r = threadIdx.x / GN, rem = threadIdx.x - r * GN, g = rem / N, n = rem - g * N;
    const int ridx = blockIdx.x * rpc + r;
    const bool valid = (r < rpc) && (ridx < a.nn);
    int A = ridx, kb = 0, ke = 0;
    if (valid) {
        if (a.rows) {
            const int4 rr = __ldg(a.rows + ridx);
            A = rr.x;
            kb = rr.y;
            ke = rr.z;
        } else {
            A = a.perm ? __ldg(a.perm + ridx) : ridx;
            kb = __ldg(a.row_ptr + A);
            ke = __ldg(a.row_ptr + A + 1);
        }
    }
    double acc[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // ou0 ou1 ou2 op t0 t1 t2
    if (valid) {
        const long N8 = 8L * N;
        int Bn = kb + g < ke ? __ldg(a.col_idx + kb + g) : 0;
#pragma unroll 2
        for (int k = kb + g; k < ke; k += G) {
            const int B = Bn;
            Bn = k + G < ke ? __ldg(a.col_idx + k + G) : 0;
            const double* v = a.vals + (long)k * N8 + n;
            const long yb = (long)B * 4 * N + n;
            const double y0 = __ldg(a.y + yb), y1 = __ldg(a.y + yb + N), y2 = __ldg(a.y + yb + 2 * N),
                         y3 = __ldg(a.y + yb + 3 * N);
            const double kd = ldcs(v), g0 = ldcs(v + N), g1 = ldcs(v + 2 * N), g2 = ldcs(v + 3 * N);
            const double d0 = ldcs(v + 4 * N), d1 = ldcs(v + 5 * N), d2 = ldcs(v + 6 * N), ld = ldcs(v + 7 * N);
            acc[0] += kd * y0 + g0 * y3;
            acc[1] += kd * y1 + g1 * y3;
            acc[2] += kd * y2 + g2 * y3;
            acc[3] += d0 * y0;
            acc[3] += d1 * y1;
            acc[3] += d2 * y2;
            acc[3] += ld * y3;
            if (WITH_C) {
                const double m = __ldg(a.mass + k);
                acc[4] += m * y0;
                acc[5] += m * y1;
                acc[6] += m * y2;
            }
        }
    }
    constexpr int NV = WITH_C ? 7 : 4;
    if (valid) {
        double* p = pr + ((size_t)(r * G + g) * 7) * N + n;
#pragma unroll
        for (int c = 0; c < NV; ++c)
            p[c * N] = acc[c];
    }
    __syncthreads();
    const bool lead = valid && g == 0;
    if (lead) {
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            double v = 0.0;
            for (int gg = 0; gg < G; ++gg)
                v += pr[((size_t)(r * G + gg) * 7 + c) * N + n];
            acc[c] = v;
        }
    }
    if (WITH_C) {
        if (lead) {
            st[(r * 3 + 0) * N + n] = acc[4];
            st[(r * 3 + 1) * N + n] = acc[5];
            st[(r * 3 + 2) * N + n] = acc[6];
        }
        __syncthreads();
        if (lead) {
            const double* h = sH + n * N;
            const double* s0 = st + (r * 3) * N;
            double h0 = 0.0, h1 = 0.0, h2 = 0.0;
            for (int m = 0; m < N; ++m) {
                const double hm = h[m];
                h0 += hm * s0[m];
                h1 += hm * s0[N + m];
                h2 += hm * s0[2 * N + m];
            }
            acc[0] += h0;
            acc[1] += h1;
            acc[2] += h2;
        }
    }
    if (lead) {
        const long o = (long)A * 4 * N + n;
        if (SCALED) {
            acc[0] *= __ldg(a.scale_out + o);
            acc[1] *= __ldg(a.scale_out + o + N);
            acc[2] *= __ldg(a.scale_out + o + 2 * N);
            acc[3] *= __ldg(a.scale_out + o + 3 * N);
        }
        a.out[o] = acc[0];
        a.out[o + N] = acc[1];
        a.out[o + 2 * N] = acc[2];
        a.out[o + 3 * N] = acc[3];
    }
}

template <int G>
static void launch_lmatvec_g(const MatvecArgs& a_in, cudaStream_t st) {
    MatvecArgs a = a_in;
    a.rows_per_cta = max(1, 256 / (G * a.N));
    const int blocks = (a.nn + a.rows_per_cta - 1) / a.rows_per_cta;
    const int threads = a.rows_per_cta * G * a.N;
    const bool wc = a.with_c != 0;
    const size_t smem = sizeof(double) * ((wc ? (size_t)a.N * a.N + 3 * (size_t)a.N * a.rows_per_cta : 0) +
                                          7 * (size_t)G * a.N * a.rows_per_cta);
    note_launch();
    if (wc) {
        if (a.scale_out)
            lmatvec_g_kernel<true, true, G><<<blocks, threads, smem, st>>>(a);
        else
            lmatvec_g_kernel<false, true, G><<<blocks, threads, smem, st>>>(a);
    } else {
        if (a.scale_out)
            lmatvec_g_kernel<true, false, G><<<blocks, threads, smem, st>>>(a);
        else
            lmatvec_g_kernel<false, false, G><<<blocks, threads, smem, st>>>(a);
    }
}

// N == 1 with G lanes per row: lane g takes blocks kb+g, kb+g+G, ... (64-byte
// blocks as four 16-byte loads), the G partial sums are combined by a fixed
// xor-shuffle tree (deterministic).  Rows are taken in `perm` order.
template <bool SCALED, int G>
__global__ void __launch_bounds__(256) lmatvec_n1g_kernel(MatvecArgs a) {
    if (a.skip && *a.skip)
        return;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int ridx = t / G, g = t & (G - 1);
    const bool valid = ridx < a.nn;
    int A = 0, kb = 0, ke = 0;
    if (valid) {
        if (a.rows) {
            const int4 rr = __ldg(a.rows + ridx);
            A = rr.x;
            kb = rr.y;
            ke = rr.z;
        } else {
            A = a.perm ? __ldg(a.perm + ridx) : ridx;
            kb = __ldg(a.row_ptr + A);
            ke = __ldg(a.row_ptr + A + 1);
        }
    }
    double ou0 = 0.0, ou1 = 0.0, ou2 = 0.0, op = 0.0;
    if (valid) {
#pragma unroll 2
        for (int k = kb + g; k < ke; k += G) {
            const int B = __ldg(&a.col_idx[k]);
            const double2* v = reinterpret_cast<const double2*>(a.vals + (long)k * 8);
            const double2* yv = reinterpret_cast<const double2*>(a.y + (long)B * 4);
            const double2 ya = __ldg(yv), yb = __ldg(yv + 1);
            const double2 p0 = ldcs2(v), p1 = ldcs2(v + 1), p2 = ldcs2(v + 2), p3 = ldcs2(v + 3);
            ou0 += p0.x * ya.x + p0.y * yb.y;
            ou1 += p0.x * ya.y + p1.x * yb.y;
            ou2 += p0.x * yb.x + p1.y * yb.y;
            op += p2.x * ya.x;
            op += p2.y * ya.y;
            op += p3.x * yb.x;
            op += p3.y * yb.y;
        }
    }
#pragma unroll
    for (int off = 1; off < G; off <<= 1) {
        ou0 += __shfl_xor_sync(0xffffffffu, ou0, off, G);
        ou1 += __shfl_xor_sync(0xffffffffu, ou1, off, G);
        ou2 += __shfl_xor_sync(0xffffffffu, ou2, off, G);
        op += __shfl_xor_sync(0xffffffffu, op, off, G);
    }
    if (valid && g == 0) {
        const long o = (long)A * 4;
        if (SCALED) {
            const double2 s0 = __ldg(reinterpret_cast<const double2*>(a.scale_out + o));
            const double2 s1 = __ldg(reinterpret_cast<const double2*>(a.scale_out + o) + 1);
            ou0 *= s0.x;
            ou1 *= s0.y;
            ou2 *= s1.x;
            op *= s1.y;
        }
        double2* out = reinterpret_cast<double2*>(a.out + o);
        out[0] = make_double2(ou0, ou1);
        out[1] = make_double2(ou2, op);
    }
}

void launch_lmatvec(const MatvecArgs& a_in, cudaStream_t st) {
    if (a_in.nn <= 0)
        return;
    MatvecArgs a = a_in;
    // Rows in the length-balanced order as {A, kb, ke} records.  N == 1: four
    // lanes per row (config 4: 0.277 -> 0.189 ms).  N > 1: four lanes per
    // (row, sample) when the (row, sample) threads alone cannot fill the GPU
    // (config 0: 26.7 -> 18.5 us; on the large meshes the split costs 35-40%).
    if (a.N == 1) {
        constexpr int G = 4;
        const int blocks = (int)(((long)a.nn * G + 255) / 256);
        note_launch();
        if (a.scale_out)
            lmatvec_n1g_kernel<true, G><<<blocks, 256, 0, st>>>(a);
        else
            lmatvec_n1g_kernel<false, G><<<blocks, 256, 0, st>>>(a);
        return;
    }
    const bool split = a.lanes == 4 || (a.lanes == 0 && (long)a.nn * a.N < 65536);
    if (split)
        return launch_lmatvec_g<4>(a, st);
    const int blocks = (a.nn + a.rows_per_cta - 1) / a.rows_per_cta;
    const int threads = a.rows_per_cta * a.N;
    const size_t smem =
        a.with_c ? sizeof(double) * ((size_t)a.N * a.N + 3 * (size_t)a.N * a.rows_per_cta) : 0;
    note_launch();
    launch_main(a, blocks, threads, smem, st);
}

// mass_c[k] = mass[k] unless the row or the column node is Dirichlet
// (the C-part masking of linalg.cpp:109,115).
__global__ void mask_mass_kernel(const double* __restrict__ mass, const int* __restrict__ row_ptr,
                                 const int* __restrict__ col_idx, const uint8_t* __restrict__ dir,
                                 int nn, double* __restrict__ mass_c) {
    const int A = blockIdx.x * blockDim.x + threadIdx.x;
    if (A >= nn)
        return;
    const bool af = dir[A] != 0;
    for (int k = row_ptr[A]; k < row_ptr[A + 1]; ++k)
        mass_c[k] = (af || dir[col_idx[k]]) ? 0.0 : mass[k];
}

void launch_mask_mass(const double* mass, const int* row_ptr, const int* col_idx,
                      const uint8_t* dir, int nn, double* mass_c, cudaStream_t st) {
    if (nn <= 0)
        return;
    note_launch();
    mask_mass_kernel<<<(nn + 255) / 256, 256, 0, st>>>(mass, row_ptr, col_idx, dir, nn, mass_c);
}

}  // namespace hbgpu
