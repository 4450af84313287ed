// Pointwise tangent P and consistent mass, row-owned (sm_100a, FP64).
//
// Replaces element_tangent_p + assemble_tangent (reference
// src/assembly.cpp:265-374, 550-666) and assemble_mass (:668-681).
#include "hbgpu_internal.h"

namespace hbgpu {

namespace {
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace

// Compact per-element geometry for the tangent: gradN[4][3], V, symmetric xi
// (00 01 02 11 12 22), xi:xi  -> 20 doubles, 16-byte aligned records.
__global__ void tangent_geometry_kernel(const double* __restrict__ geom, int ne,
                                        double* __restrict__ tg) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne)
        return;
    const double* g = geom + 22 * (long)e;
    double* o = tg + kTGeo * (long)e;
    for (int k = 0; k < 13; ++k)
        o[k] = g[k];
    o[13] = g[13];
    o[14] = g[14];
    o[15] = g[15];
    o[16] = g[17];
    o[17] = g[18];
    o[18] = g[21];
    double s = 0.0;
    for (int k = 0; k < 9; ++k)
        s += g[13 + k] * g[13 + k];
    o[19] = s;
}

void launch_tangent_geometry(const double* geom, int ne, double* tg, cudaStream_t st) {
    if (ne <= 0)
        return;
    note_launch();
    tangent_geometry_kernel<<<(ne + 255) / 256, 256, 0, st>>>(geom, ne, tg);
}

namespace {

struct IncData {
    double g[kTGeo];
    double u[4][3];
};

__device__ __forceinline__ void fetch_inc(const TangentArgs& a, const int4 r0, const int4 r1, int n,
                                          IncData& d) {
    const int e = r1.x & 0x3FFFFFFF;
    const double2* g2 = reinterpret_cast<const double2*>(a.tgeom + (long)kTGeo * e);
#pragma unroll
    for (int k = 0; k < kTGeo / 2; ++k) {
        const double2 v = __ldg(g2 + k);
        d.g[2 * k] = v.x;
        d.g[2 * k + 1] = v.y;
    }
    const int nd[4] = {r0.x, r0.y, r0.z, r0.w};
    const int N = a.N;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const double* sb = a.state + (long)nd[b] * 4 * N + n;
#pragma unroll
        for (int i = 0; i < 3; ++i)
            d.u[b][i] = __ldg(sb + i * N);
    }
}

__device__ __forceinline__ double xi_quad(const double* g, const double u[3]) {
    // u . xi u with the symmetric xi of the compact record
    return g[13] * u[0] * u[0] + g[16] * u[1] * u[1] + g[18] * u[2] * u[2] +
           2.0 * (g[14] * u[0] * u[1] + g[15] * u[0] * u[2] + g[17] * u[1] * u[2]);
}

}  // namespace

// Row-owned assembly of P.  A CTA owns `rows` consecutive block rows; its
// shared memory holds exactly their P.vals segment ([blk][slot][n], the
// global layout), accumulated on chip and written once, coalesced.  Thread
// (row A, sample n) walks the elements containing A in element order — the
// reference's summation order per block — and adds each element's
// contribution to the 4 blocks (A, conn[e][b]).  Incidence records are
// prefetched two ahead and their geometry / velocities one ahead, so global
// latency overlaps the FP64 work of the current element.
//
// Per element and sample the quadrature sums factor through 8 scalars:
//   K_ab = kc_ab + kappa_a . gradN_b,  kappa_a = w rho sum_q (N_a(q) + tau_q adv_a(q)) u_q
//   G_ab = -dN_a V/4 + alpha_a gradN_b, alpha_a = w sum_q tau_q adv_a(q)
//   D_ab = dN_b V/4 + dN_a (w z . gradN_b), z = sum_q tau_q u_q
//   L_ab = gradN_a.gradN_b * (w/rho) sum_q tau_q
// (Picard-frozen tangent of assembly.cpp:265-374; masking of :583-607.)
template <int TAU>
__global__ void __launch_bounds__(128) tangent_rows_kernel(TangentArgs a) {
    extern __shared__ double sm[];
    const int N = a.N;
    const int row_lo = a.cta_rows[blockIdx.x], row_hi = a.cta_rows[blockIdx.x + 1];
    const long blk_lo = a.row_ptr[row_lo];
    const long nvals = ((long)a.row_ptr[row_hi] - blk_lo) * 8 * N;
    for (long k = threadIdx.x; k < nvals; k += blockDim.x)
        sm[k] = 0.0;
    __syncthreads();

    const int r = threadIdx.x / N, n = threadIdx.x - r * N;
    const int A = row_lo + r;
    if (A < row_hi) {
        const long rowoff = (long)a.row_ptr[A] - blk_lo;
        const double rho = a.rho, diffc = 3.0 * a.nu * a.nu;
        const int i0 = a.inc_ptr[A], i1 = a.inc_ptr[A + 1];
        const int4* rec = a.inc_rec;
        int4 c0 = make_int4(0, 0, 0, 0), c1 = c0, n0 = c0, n1 = c0;
        IncData cur, nxt;
        if (i0 < i1) {
            c0 = __ldg(rec + 2 * i0);
            c1 = __ldg(rec + 2 * i0 + 1);
            if (i0 + 1 < i1) {
                n0 = __ldg(rec + 2 * i0 + 2);
                n1 = __ldg(rec + 2 * i0 + 3);
            }
            fetch_inc(a, c0, c1, n, cur);
        }
        long diag_local = -1;
        for (int ii = i0; ii < i1; ++ii) {
            int4 m0 = make_int4(0, 0, 0, 0), m1 = m0;
            if (ii + 2 < i1) {
                m0 = __ldg(rec + 2 * ii + 4);
                m1 = __ldg(rec + 2 * ii + 5);
            }
            if (ii + 1 < i1)
                fetch_inc(a, n0, n1, n, nxt);

            const int la = (unsigned)c1.x >> 30;
            const unsigned cols = (unsigned)c1.y;
            const int em = c1.z;
            const double* g = cur.g;
            const double V = g[12], w = 0.25 * V;
            double usum[3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
                usum[i] = cur.u[0][i] + cur.u[1][i] + cur.u[2][i] + cur.u[3][i];
            const double diff = diffc * g[19];
            double tau_mean = 0.0;
            if (TAU == 1) {
                const double um[3] = {0.25 * usum[0], 0.25 * usum[1], 0.25 * usum[2]};
                const double arg = xi_quad(g, um) + diff;
                if (!(arg > 0.0))
                    atomicOr(a.flag, 1);
                tau_mean = arg > 0.0 ? rsqrt(arg) : 0.0;
            }
            double ga[3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
                ga[i] = la == 0 ? g[i] : la == 1 ? g[3 + i] : la == 2 ? g[6 + i] : g[9 + i];
            double asum = 0.0, tsum = 0.0, z[3] = {0.0, 0.0, 0.0}, kap[3] = {0.0, 0.0, 0.0};
            const double dAB = kQA - kQB;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double uq[3];
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    uq[i] = kQB * usum[i] + dAB * cur.u[q][i];
                double tq = tau_mean;
                if (TAU == 0) {
                    const double arg = xi_quad(g, uq) + diff;
                    if (!(arg > 0.0))
                        atomicOr(a.flag, 1);
                    tq = arg > 0.0 ? rsqrt(arg) : 0.0;
                }
                const double tadv = tq * (uq[0] * ga[0] + uq[1] * ga[1] + uq[2] * ga[2]);
                const double na = (q == la) ? kQA : kQB;
                asum += tadv;
                tsum += tq;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    z[i] += tq * uq[i];
                    kap[i] += (na + tadv) * uq[i];
                }
            }
            const double alpha_a = w * asum, beta = (w / rho) * tsum, wr = w * rho;
            const bool afix = (em >> la) & 1;
            const double muV = a.mu * V, pcV = a.pseudo_c * V;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int j = (cols >> (8 * b)) & 0xFF;
                double* acc = sm + (rowoff + j) * 8 * N + n;
                const bool bfix = (em >> b) & 1;
                const double* gb = g + 3 * b;
                const double gg = ga[0] * gb[0] + ga[1] * gb[1] + ga[2] * gb[2];
                if (!afix && !bfix) {
                    const double kc = muV * gg + pcV * (b == la ? 0.1 : 0.05);
                    acc[0] += kc + wr * (kap[0] * gb[0] + kap[1] * gb[1] + kap[2] * gb[2]);
                }
                if (!afix) {
#pragma unroll
                    for (int i = 0; i < 3; ++i)
                        acc[(1 + i) * N] += -ga[i] * w + alpha_a * gb[i];
                }
                if (!bfix) {
                    const double alpha_b = w * (z[0] * gb[0] + z[1] * gb[1] + z[2] * gb[2]);
#pragma unroll
                    for (int i = 0; i < 3; ++i)
                        acc[(4 + i) * N] += gb[i] * w + ga[i] * alpha_b;
                }
                acc[7 * N] += gg * beta;
                if (b == la)
                    diag_local = rowoff + j;
            }
            c0 = n0;
            c1 = n1;
            n0 = m0;
            n1 = m1;
            cur = nxt;
        }
        // identity on constrained velocity diagonals (assembly.cpp:659-665)
        if (a.dir[A] && diag_local >= 0)
            sm[diag_local * 8 * N + n] = 1.0;
    }
    __syncthreads();
    const double2* s2 = reinterpret_cast<const double2*>(sm);
    double2* d2 = reinterpret_cast<double2*>(a.pvals + blk_lo * 8 * N);
    for (long k = threadIdx.x; k < nvals / 2; k += blockDim.x)
        d2[k] = s2[k];
}

// ---------------------------------------------------------------------------
// Tangent v3: one CTA per block row A, two phases.
//  Phase 1 — every (incidence i, sample n) pair of the row computes its
//    element summary in parallel into shared memory:
//      kappa_a (3) = w rho sum_q (N_a(q) + tau_q adv_a(q)) u_q,  alpha_a,
//      z (3) = sum_q tau_q u_q,  beta = (w/rho) sum_q tau_q
//    (and the element's gradN, V for phase 2).
//  Phase 2 — every (block j of the row, sample n) accumulates its
//    contributions (i, b) in element order in registers and writes the 8
//    slots of P.vals once:
//      K += mu V gg + pc V m_ab + kappa_a . gradN_b,  G_i += -dN_a,i w + alpha_a dN_b,i
//      D_i += dN_b,i w + dN_a,i (w z . gradN_b),       L += gg beta
//    The diagonal block (all ~24 incidences) is split into parts of <= 8
//    contributions summed in fixed order, so the threads stay balanced.
// Masks (assembly.cpp:583-607) are per block: afix = dir[A], bfix = dir[B].
template <int TAU>
__global__ void __launch_bounds__(kTanThreads, TAN_MINB) tangent_row_kernel(TangentArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int N = a.N;
    const int A = a.rows[blockIdx.x];  // rows are bucketed by valence
    // time-sample tile of this CTA (all N unless a high-valence row at large
    // N would overflow shared memory)
    const int NT = a.NT, n0 = blockIdx.y * NT, nt = min(NT, N - n0);
    const int i0 = a.inc_ptr[A], ninc = a.inc_ptr[A + 1] - i0;
    const int k0 = a.row_ptr[A], nblk = a.row_ptr[A + 1] - k0;
    double* summ = sm;                                   // [i][8][t]
    double* geo = summ + (size_t)a.max_inc * 8 * NT;     // [i][16]: gradN 12, V, la
    double* dpart = geo + (size_t)a.max_inc * 16;        // [part][8][t] diagonal partials
    const double rho = a.rho, diffc = 3.0 * a.nu * a.nu, dAB = kQA - kQB;

    for (int it = threadIdx.x; it < ninc * nt; it += blockDim.x) {
        const int i = it / nt, t = it - i * nt, n = n0 + t;
        const int4 r0 = __ldg(a.inc_rec + 2 * (i0 + i));
        const int4 r1 = __ldg(a.inc_rec + 2 * (i0 + i) + 1);
        const int e = r1.x & 0x3FFFFFFF, la = (unsigned)r1.x >> 30;
        const double* g = a.tgeom + (long)kTGeo * e;
        if (t == 0) {
            for (int k = 0; k < 13; ++k)
                geo[i * 16 + k] = __ldg(g + k);
            geo[i * 16 + 13] = double(la);
        }
        const int nd[4] = {r0.x, r0.y, r0.z, r0.w};
        double u[4][3], usum[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double* sb = a.state + (long)nd[b] * 4 * N + n;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                u[b][c] = __ldg(sb + c * N);
                usum[c] += u[b][c];
            }
        }
        double xs[7];
#pragma unroll
        for (int k = 0; k < 7; ++k)
            xs[k] = __ldg(g + 13 + k);  // xi00 xi01 xi02 xi11 xi12 xi22 xi:xi
        const double V = __ldg(g + 12), w = 0.25 * V, diff = diffc * xs[6];
        double ga[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            ga[c] = __ldg(g + 3 * la + c);
        auto quad = [&](const double v[3]) {
            return xs[0] * v[0] * v[0] + xs[3] * v[1] * v[1] + xs[5] * v[2] * v[2] +
                   2.0 * (xs[1] * v[0] * v[1] + xs[2] * v[0] * v[2] + xs[4] * v[1] * v[2]);
        };
        double tau_mean = 0.0;
        if (TAU == 1) {
            const double um[3] = {0.25 * usum[0], 0.25 * usum[1], 0.25 * usum[2]};
            const double arg = quad(um) + diff;
            if (!(arg > 0.0))
                atomicOr(a.flag, 1);
            tau_mean = arg > 0.0 ? rsqrt(arg) : 0.0;
        }
        double asum = 0.0, tsum = 0.0, z[3] = {0.0, 0.0, 0.0}, kap[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double uq[3];
#pragma unroll
            for (int c = 0; c < 3; ++c)
                uq[c] = kQB * usum[c] + dAB * u[q][c];
            double tq = tau_mean;
            if (TAU == 0) {
                const double arg = quad(uq) + diff;
                if (!(arg > 0.0))
                    atomicOr(a.flag, 1);
                tq = arg > 0.0 ? rsqrt(arg) : 0.0;
            }
            const double tadv = tq * (uq[0] * ga[0] + uq[1] * ga[1] + uq[2] * ga[2]);
            const double na = (q == la) ? kQA : kQB;
            asum += tadv;
            tsum += tq;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                z[c] += tq * uq[c];
                kap[c] += (na + tadv) * uq[c];
            }
        }
        double* s = summ + (size_t)i * 8 * NT + t;
        const double wr = w * rho;
        s[0] = wr * kap[0];
        s[NT] = wr * kap[1];
        s[2 * NT] = wr * kap[2];
        s[3 * NT] = w * asum;
        s[4 * NT] = w * z[0];
        s[5 * NT] = w * z[1];
        s[6 * NT] = w * z[2];
        s[7 * NT] = (w / rho) * tsum;
    }
    __syncthreads();

    const bool afix = a.dir[A] != 0;
    const int kdiag = a.diag_blk[A] - k0;
    const int cb = a.contrib_ptr[k0];
    const int ndiag = a.contrib_ptr[k0 + kdiag + 1] - a.contrib_ptr[k0 + kdiag];
    const int dparts = (ndiag + kTanPart - 1) / kTanPart;
    const int nitems = (nblk - 1 + dparts) * nt;
    for (int it = threadIdx.x; it < nitems; it += blockDim.x) {
        const int slot = it / nt, t = it - slot * nt, n = n0 + t;
        int j, c0, c1, part = -1;
        if (slot < nblk - 1) {
            j = slot < kdiag ? slot : slot + 1;
            c0 = a.contrib_ptr[k0 + j];
            c1 = a.contrib_ptr[k0 + j + 1];
        } else {
            j = kdiag;
            part = slot - (nblk - 1);
            c0 = a.contrib_ptr[k0 + j] + part * kTanPart;
            c1 = min(c0 + kTanPart, a.contrib_ptr[k0 + j + 1]);
        }
        const bool bfix = a.dir[a.col_idx[k0 + j]] != 0;
        double K = 0.0, G0 = 0.0, G1 = 0.0, G2 = 0.0, D0 = 0.0, D1 = 0.0, D2 = 0.0, L = 0.0;
        for (int q = c0; q < c1; ++q) {
            const int ent = a.contrib[q];
            const int i = ent >> 2, b = ent & 3;
            const double* gi = geo + i * 16;
            const int la = int(gi[13]);
            const double ga0 = gi[3 * la], ga1 = gi[3 * la + 1], ga2 = gi[3 * la + 2];
            const double gb0 = gi[3 * b], gb1 = gi[3 * b + 1], gb2 = gi[3 * b + 2];
            const double V = gi[12], w = 0.25 * V;
            const double* s = summ + (size_t)i * 8 * NT + t;
            const double gg = ga0 * gb0 + ga1 * gb1 + ga2 * gb2;
            K += a.mu * V * gg + a.pseudo_c * V * (b == la ? 0.1 : 0.05) +
                 (s[0] * gb0 + s[NT] * gb1 + s[2 * NT] * gb2);
            const double al = s[3 * NT];
            G0 += -ga0 * w + al * gb0;
            G1 += -ga1 * w + al * gb1;
            G2 += -ga2 * w + al * gb2;
            const double alb = s[4 * NT] * gb0 + s[5 * NT] * gb1 + s[6 * NT] * gb2;
            D0 += gb0 * w + ga0 * alb;
            D1 += gb1 * w + ga1 * alb;
            D2 += gb2 * w + ga2 * alb;
            L += gg * s[7 * NT];
        }
        if (afix || bfix)
            K = 0.0;
        if (afix)
            G0 = G1 = G2 = 0.0;
        if (bfix)
            D0 = D1 = D2 = 0.0;
        if (part < 0) {
            // streaming stores: P.vals must not evict the state / geometry from L2
            double* out = a.pvals + ((long)(k0 + j) * 8) * N + n;
            __stcs(out, K);
            __stcs(out + N, G0);
            __stcs(out + 2 * N, G1);
            __stcs(out + 3 * N, G2);
            __stcs(out + 4 * N, D0);
            __stcs(out + 5 * N, D1);
            __stcs(out + 6 * N, D2);
            __stcs(out + 7 * N, L);
        } else {
            double* o = dpart + (size_t)part * 8 * NT + t;
            o[0] = K;
            o[NT] = G0;
            o[2 * NT] = G1;
            o[3 * NT] = G2;
            o[4 * NT] = D0;
            o[5 * NT] = D1;
            o[6 * NT] = D2;
            o[7 * NT] = L;
        }
    }
    (void)cb;
    __syncthreads();
    // diagonal block: sum the parts in order; identity K on Dirichlet rows (assembly.cpp:659-665)
    for (int it = threadIdx.x; it < 8 * nt; it += blockDim.x) {
        const int sl = it / nt, t = it - sl * nt, n = n0 + t;
        double v = 0.0;
        for (int p = 0; p < dparts; ++p)
            v += dpart[((size_t)p * 8 + sl) * NT + t];
        if (sl == 0 && afix)
            v = 1.0;
        __stcs(a.pvals + ((long)(k0 + kdiag) * 8 + sl) * N + n, v);
    }
}

// Tangent v4 = v3 with a staging phase: before any FP64 work the CTA pulls
// everything its row needs into shared memory with cp.async — the velocities
// of the row's column nodes (the only nodes its elements touch), the compact
// geometry and the records of its elements — so phases 1 and 2 run on
// shared-memory operands only and the global latency is paid once per row,
// in bulk, overlapped with the other resident rows.
namespace {
__device__ __forceinline__ void cpa8(double* dst, const double* src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cpa16(void* dst, const void* src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cpa_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
}
}  // namespace

template <int TAU>
__global__ void __launch_bounds__(kTanThreads, TAN_MINB) tangent_row4_kernel(TangentArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int N = a.N;
    const int A = a.rows[blockIdx.x];
    const int NT = a.NT, n0 = blockIdx.y * NT, nt = min(NT, N - n0);
    const int i0 = a.inc_ptr[A], ninc = a.inc_ptr[A + 1] - i0;
    const int k0 = a.row_ptr[A], nblk = a.row_ptr[A + 1] - k0;
    double* summ = sm;                                    // [i][8][t]
    double* geo = summ + (size_t)a.max_inc * 8 * NT;      // [i][kTGeo]
    double* dpart = geo + (size_t)a.max_inc * kTGeo;      // [part][8][t]
    double* us = dpart + (size_t)((a.max_inc + kTanPart - 1) / kTanPart) * 8 * NT;  // [j][3][t]
    int4* rec = reinterpret_cast<int4*>(us + ((size_t)a.max_blk * 3 * NT + 1) / 2 * 2);  // [i]

    // ---- phase 0: stage records, geometry and column-node velocities
    for (int i = threadIdx.x; i < ninc; i += blockDim.x) {
        const int4 r1 = __ldg(a.inc_rec + 2 * (i0 + i) + 1);
        rec[i] = r1;
        const double* g = a.tgeom + (long)kTGeo * (r1.x & 0x3FFFFFFF);
#pragma unroll
        for (int k = 0; k < kTGeo / 2; ++k)
            cpa16(geo + i * kTGeo + 2 * k, g + 2 * k);
    }
    for (int it = threadIdx.x; it < nblk * 3 * nt; it += blockDim.x) {
        const int j = it / (3 * nt), rem = it - j * 3 * nt, c = rem / nt, t = rem - c * nt;
        const long B = __ldg(a.col_idx + k0 + j);
        cpa8(us + (j * 3 + c) * NT + t, a.state + (B * 4 + c) * N + n0 + t);
    }
    cpa_wait_all();
    __syncthreads();

    // ---- phase 1: element summaries per (incidence, sample)
    const double rho = a.rho, diffc = 3.0 * a.nu * a.nu, dAB = kQA - kQB;
    for (int it = threadIdx.x; it < ninc * nt; it += blockDim.x) {
        const int i = it / nt, t = it - i * nt;
        const int4 r1 = rec[i];
        const int la = (unsigned)r1.x >> 30;
        const unsigned cols = (unsigned)r1.y;
        const double* g = geo + i * kTGeo;
        double u[4][3], usum[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double* ub = us + ((cols >> (8 * b)) & 0xFF) * 3 * NT + t;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                u[b][c] = ub[c * NT];
                usum[c] += u[b][c];
            }
        }
        const double V = g[12], w = 0.25 * V, diff = diffc * g[19];
        const double ga[3] = {g[3 * la], g[3 * la + 1], g[3 * la + 2]};
        auto quad = [&](const double v[3]) {
            return g[13] * v[0] * v[0] + g[16] * v[1] * v[1] + g[18] * v[2] * v[2] +
                   2.0 * (g[14] * v[0] * v[1] + g[15] * v[0] * v[2] + g[17] * v[1] * v[2]);
        };
        double tau_mean = 0.0;
        if (TAU == 1) {
            const double um[3] = {0.25 * usum[0], 0.25 * usum[1], 0.25 * usum[2]};
            const double arg = quad(um) + diff;
            if (!(arg > 0.0))
                atomicOr(a.flag, 1);
            tau_mean = arg > 0.0 ? rsqrt(arg) : 0.0;
        }
        double asum = 0.0, tsum = 0.0, z[3] = {0.0, 0.0, 0.0}, kap[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double uq[3];
#pragma unroll
            for (int c = 0; c < 3; ++c)
                uq[c] = kQB * usum[c] + dAB * u[q][c];
            double tq = tau_mean;
            if (TAU == 0) {
                const double arg = quad(uq) + diff;
                if (!(arg > 0.0))
                    atomicOr(a.flag, 1);
                tq = arg > 0.0 ? rsqrt(arg) : 0.0;
            }
            const double tadv = tq * (uq[0] * ga[0] + uq[1] * ga[1] + uq[2] * ga[2]);
            const double na = (q == la) ? kQA : kQB;
            asum += tadv;
            tsum += tq;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                z[c] += tq * uq[c];
                kap[c] += (na + tadv) * uq[c];
            }
        }
        double* s = summ + (size_t)i * 8 * NT + t;
        const double wr = w * rho;
        s[0] = wr * kap[0];
        s[NT] = wr * kap[1];
        s[2 * NT] = wr * kap[2];
        s[3 * NT] = w * asum;
        s[4 * NT] = w * z[0];
        s[5 * NT] = w * z[1];
        s[6 * NT] = w * z[2];
        s[7 * NT] = (w / rho) * tsum;
    }
    __syncthreads();

    // ---- phase 2: blocks accumulate their contributions in element order
    const bool afix = a.dir[A] != 0;
    const int kdiag = a.diag_blk[A] - k0;
    const int ndiag = a.contrib_ptr[k0 + kdiag + 1] - a.contrib_ptr[k0 + kdiag];
    const int dparts = (ndiag + kTanPart - 1) / kTanPart;
    const int nitems = (nblk - 1 + dparts) * nt;
    const double muc = a.mu, pcc = a.pseudo_c;
    for (int it = threadIdx.x; it < nitems; it += blockDim.x) {
        const int slot = it / nt, t = it - slot * nt, n = n0 + t;
        int j, c0, c1, part = -1;
        if (slot < nblk - 1) {
            j = slot < kdiag ? slot : slot + 1;
            c0 = a.contrib_ptr[k0 + j];
            c1 = a.contrib_ptr[k0 + j + 1];
        } else {
            j = kdiag;
            part = slot - (nblk - 1);
            c0 = a.contrib_ptr[k0 + j] + part * kTanPart;
            c1 = min(c0 + kTanPart, a.contrib_ptr[k0 + j + 1]);
        }
        const bool bfix = a.dir[a.col_idx[k0 + j]] != 0;
        double K = 0.0, G0 = 0.0, G1 = 0.0, G2 = 0.0, D0 = 0.0, D1 = 0.0, D2 = 0.0, L = 0.0;
        for (int q = c0; q < c1; ++q) {
            const int ent = a.contrib[q];
            const int i = ent >> 2, b = ent & 3;
            const double* gi = geo + i * kTGeo;
            const int la = (unsigned)rec[i].x >> 30;
            const double ga0 = gi[3 * la], ga1 = gi[3 * la + 1], ga2 = gi[3 * la + 2];
            const double gb0 = gi[3 * b], gb1 = gi[3 * b + 1], gb2 = gi[3 * b + 2];
            const double V = gi[12], w = 0.25 * V;
            const double* s = summ + (size_t)i * 8 * NT + t;
            const double gg = ga0 * gb0 + ga1 * gb1 + ga2 * gb2;
            K += muc * V * gg + pcc * V * (b == la ? 0.1 : 0.05) +
                 (s[0] * gb0 + s[NT] * gb1 + s[2 * NT] * gb2);
            const double al = s[3 * NT];
            G0 += -ga0 * w + al * gb0;
            G1 += -ga1 * w + al * gb1;
            G2 += -ga2 * w + al * gb2;
            const double alb = s[4 * NT] * gb0 + s[5 * NT] * gb1 + s[6 * NT] * gb2;
            D0 += gb0 * w + ga0 * alb;
            D1 += gb1 * w + ga1 * alb;
            D2 += gb2 * w + ga2 * alb;
            L += gg * s[7 * NT];
        }
        if (afix || bfix)
            K = 0.0;
        if (afix)
            G0 = G1 = G2 = 0.0;
        if (bfix)
            D0 = D1 = D2 = 0.0;
        double* o;
        long st;
        if (part < 0) {
            o = a.pvals + ((long)(k0 + j) * 8) * N + n;
            st = N;
            __stcs(o, K);
            __stcs(o + st, G0);
            __stcs(o + 2 * st, G1);
            __stcs(o + 3 * st, G2);
            __stcs(o + 4 * st, D0);
            __stcs(o + 5 * st, D1);
            __stcs(o + 6 * st, D2);
            __stcs(o + 7 * st, L);
        } else {
            o = dpart + (size_t)part * 8 * NT + t;
            o[0] = K;
            o[NT] = G0;
            o[2 * NT] = G1;
            o[3 * NT] = G2;
            o[4 * NT] = D0;
            o[5 * NT] = D1;
            o[6 * NT] = D2;
            o[7 * NT] = L;
        }
    }
    __syncthreads();
    for (int it = threadIdx.x; it < 8 * nt; it += blockDim.x) {
        const int sl = it / nt, t = it - sl * nt, n = n0 + t;
        double v = 0.0;
        for (int p = 0; p < dparts; ++p)
            v += dpart[((size_t)p * 8 + sl) * NT + t];
        if (sl == 0 && afix)
            v = 1.0;  // identity on constrained velocity diagonals (assembly.cpp:659-665)
        __stcs(a.pvals + ((long)(k0 + kdiag) * 8 + sl) * N + n, v);
    }
}

size_t tangent_row4_smem(int max_inc, int max_blk, int NT) {
    const int dparts = (max_inc + kTanPart - 1) / kTanPart;
    return sizeof(double) * ((size_t)max_inc * 8 * NT + (size_t)max_inc * kTGeo +
                             (size_t)dparts * 8 * NT + ((size_t)max_blk * 3 * NT + 1) / 2 * 2) +
           sizeof(int4) * (size_t)max_inc;
}

cudaError_t configure_tangent_row4_smem(size_t bytes) {
    const int b = int(bytes < 48 * 1024 ? 48 * 1024 : bytes);
    cudaError_t e = cudaFuncSetAttribute(tangent_row4_kernel<0>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e != cudaSuccess)
        return e;
    return cudaFuncSetAttribute(tangent_row4_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

void launch_tangent_row4(const TangentArgs& a, int nrows, size_t smem, cudaStream_t st) {
    if (nrows <= 0)
        return;
    note_launch();
    const dim3 grid(nrows, (a.N + a.NT - 1) / a.NT);
    if (a.tau_mode == 1)
        tangent_row4_kernel<1><<<grid, kTanThreads, smem, st>>>(a);
    else
        tangent_row4_kernel<0><<<grid, kTanThreads, smem, st>>>(a);
}

size_t tangent_row_smem(int max_inc, int max_dparts, int N) {
    return sizeof(double) * ((size_t)max_inc * 8 * N + (size_t)max_inc * 16 + (size_t)max_dparts * 8 * N);
}

cudaError_t configure_tangent_row_smem(size_t bytes) {
    const int b = int(bytes < 48 * 1024 ? 48 * 1024 : bytes);
    cudaError_t e = cudaFuncSetAttribute(tangent_row_kernel<0>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e != cudaSuccess)
        return e;
    return cudaFuncSetAttribute(tangent_row_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

void launch_tangent_row(const TangentArgs& a, int nrows, size_t smem, cudaStream_t st) {
    if (nrows <= 0)
        return;
    note_launch();
    const dim3 grid(nrows, (a.N + a.NT - 1) / a.NT);
    if (a.tau_mode == 1)
        tangent_row_kernel<1><<<grid, kTanThreads, smem, st>>>(a);
    else
        tangent_row_kernel<0><<<grid, kTanThreads, smem, st>>>(a);
}

cudaError_t configure_tangent_smem(size_t bytes) {
    const int b = int(bytes < 48 * 1024 ? 48 * 1024 : bytes);
    cudaError_t e = cudaFuncSetAttribute(tangent_rows_kernel<0>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e != cudaSuccess)
        return e;
    return cudaFuncSetAttribute(tangent_rows_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                b);
}

void launch_tangent_rows(const TangentArgs& a, int nctas, int threads, size_t smem,
                         cudaStream_t st) {
    if (nctas <= 0)
        return;
    note_launch();
    if (a.tau_mode == 1)
        tangent_rows_kernel<1><<<nctas, threads, smem, st>>>(a);
    else
        tangent_rows_kernel<0><<<nctas, threads, smem, st>>>(a);
}

// Optional frozen-coefficient backflow tangent (assembly.cpp:612-657):
// K_AB -= w N_a(q) N_b(q) (rho beta / 2) min(u_q . n, 0) for free A, B on a
// Neumann facet.  Node-centric: thread (boundary row A, n) walks A's facets in
// the reference order (Neumann entry, facet, quadrature point, b).
__global__ void backflow_tangent_kernel(BoundaryArgs a, const int* __restrict__ row_ptr,
                                        const int* __restrict__ col_idx,
                                        double* __restrict__ pvals) {
    const int N = a.N;
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int bn = (int)(t / N);
    const int n = (int)(t - (long)bn * N);
    if (bn >= a.nbnodes)
        return;
    const int A = a.bnode[bn];
    if (a.dir[A])
        return;
    const int r0 = row_ptr[A], r1 = row_ptr[A + 1];
    for (int k = a.bptr[bn]; k < a.bptr[bn + 1]; ++k) {
        const int f = a.binc[k] >> 2, v = a.binc[k] & 3;
        const int fn[3] = {a.fac[3 * f], a.fac[3 * f + 1], a.fac[3 * f + 2]};
        const double nv[3] = {a.fnormal[3 * f], a.fnormal[3 * f + 1], a.fnormal[3 * f + 2]};
        const double w = a.farea[f] / 3.0;
        double uf[3][3];
        for (int c = 0; c < 3; ++c)
            for (int i = 0; i < 3; ++i)
                uf[c][i] = a.state[((long)fn[c] * 4 + i) * N + n];
        for (int q = 0; q < 3; ++q) {
            double un = 0.0;
            for (int i = 0; i < 3; ++i) {
                double uq = 0.0;
                for (int c = 0; c < 3; ++c)
                    uq += (q == c ? 2.0 / 3.0 : 1.0 / 6.0) * uf[c][i];
                un += uq * nv[i];
            }
            if (!(un < 0.0))
                continue;
            for (int b = 0; b < 3; ++b) {
                const int B = fn[b];
                if (a.dir[B])
                    continue;
                int lo = r0, hi = r1;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (col_idx[mid] < B)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                const double c = w * (q == v ? 2.0 / 3.0 : 1.0 / 6.0) * (q == b ? 2.0 / 3.0 : 1.0 / 6.0) *
                                 0.5 * a.rho * a.beta;
                pvals[((long)lo * 8) * N + n] -= c * un;
            }
        }
    }
}

void launch_backflow_tangent(const BoundaryArgs& a, const int* row_ptr, const int* col_idx,
                             double* pvals, cudaStream_t st) {
    if (a.nbnodes <= 0)
        return;
    note_launch();
    const long threads = (long)a.nbnodes * a.N;
    backflow_tangent_kernel<<<(int)((threads + 127) / 128), 128, 0, st>>>(a, row_ptr, col_idx, pvals);
}

// assemble_mass (assembly.cpp:668-681), row-owned: each block row sums its
// elements in element order — the reference's order, hence bit-identical.
__global__ void mass_rows_kernel(const double* __restrict__ geom, const int* __restrict__ row_ptr,
                                 const int* __restrict__ inc_ptr, const int4* __restrict__ rec,
                                 double rho, double* __restrict__ mass, int nn) {
    const int A = blockIdx.x * blockDim.x + threadIdx.x;
    if (A >= nn)
        return;
    double* m = mass + row_ptr[A];
    for (int k = row_ptr[A]; k < row_ptr[A + 1]; ++k)
        mass[k] = 0.0;
    for (int ii = inc_ptr[A]; ii < inc_ptr[A + 1]; ++ii) {
        const int4 r1 = rec[2 * ii + 1];
        const int e = r1.x & 0x3FFFFFFF, la = (unsigned)r1.x >> 30;
        const unsigned cols = (unsigned)r1.y;
        const double V = geom[22 * (long)e + 12];
        const double diag = rho * V / 10.0, off = rho * V / 20.0;
        for (int b = 0; b < 4; ++b)
            m[(cols >> (8 * b)) & 0xFF] += (b == la) ? diag : off;
    }
}

void launch_mass_rows(const double* geom, const int* row_ptr, const int* inc_ptr, const int4* rec,
                      double rho, double* mass, int nn, cudaStream_t st) {
    if (nn <= 0)
        return;
    note_launch();
    mass_rows_kernel<<<(nn + 127) / 128, 128, 0, st>>>(geom, row_ptr, inc_ptr, rec, rho, mass, nn);
}

}  // namespace hbgpu
