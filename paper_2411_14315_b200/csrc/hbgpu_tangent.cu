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

// ---------------------------------------------------------------------------
// One CTA per block row A (and time-sample tile), two phases.
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
