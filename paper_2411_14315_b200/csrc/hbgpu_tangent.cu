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
// Tangent row kernel (one CTA per block row and time-sample tile): the
// fallback for rows too large for the persistent pipeline
// (hbgpu_tangent_pipe.cu), which shares its arithmetic:
//  phase 1 — every (incidence i, sample n) of the row computes the element
//    summary  kappa_a (3) = w rho sum_q (N_a(q) + tau_q u_q . dN_a) u_q,
//    w alpha_a = w sum_q tau_q u_q . dN_a,  w z (3) = w sum_q tau_q u_q,
//    beta = (w / rho) sum_q tau_q   into shared memory;
//  phase 2 — every (block slot, sample) accumulates its contributions (i, b)
//    in element order in registers and writes the 8 slots of P.vals once;
//    the diagonal block (one contribution per incidence) is split into parts
//    of kTanPart summed in fixed order.
// Masks (assembly.cpp:583-607) are per block: afix = dir[A], bfix = dir[B].
// Structure:
//  * every global load is issued in one stage (A) right after the row
//    descriptor, with dependent chains at most two loads deep, and lands in
//    shared memory: neighbour velocities su, per-incidence geometry incg,
//    the row's contribution list, per-slot metadata and block constants;
//  * the n-invariant part of every block (mu V gg + pc V m_ab, -w dN_a,
//    w dN_b summed over its contributions) is a mesh constant blkc[k][8] =
//    {sum V gg, sum V m_ab, sum -w dN_a (3), sum w dN_b (3)} computed once at
//    setup (tangent_blockconst_kernel) and added once per (block, sample);
//  * phase 2 walks per-contribution records in list order {dN_a (3), gg,
//    dN_b (3), summary offset} built from incg next to phase 1, so its inner
//    loop is 13 FMAs on shared-memory operands:
//      K += kappa . dN_b, G += alpha dN_b, D += dN_a (z . dN_b), L += gg beta;
//  * off-diagonal blocks are visited in descending contribution count
//    (blk_order) so the threads of a warp run loops of similar length.
// Row descriptor (host-built per bucket row): {A, i0, ninc, k0}, {nblk, cb, kdiag, 0}.
constexpr int kIncg = 24;  // doubles per incidence record in shared memory

struct Tan5Smem {
    int summ, su, incg, rec, scont, sinfo, sblkc, total;  // offsets in doubles
};
__host__ __device__ inline Tan5Smem tan5_layout(int mi, int max_blk, int NT) {
    Tan5Smem L;
    const int dpmax = (mi + kTanPart - 1) / kTanPart;
    int su = max_blk * 3 * NT, dp = dpmax * 8 * NT;
    su = ((su > dp ? su : dp) + 1) & ~1;  // diagonal partials reuse su after phase 1
    L.summ = 0;
    L.su = mi * 8 * NT;
    L.incg = L.su + su;
    L.rec = L.incg + mi * kIncg;
    L.scont = L.rec + mi * 32;
    L.sinfo = L.scont + ((mi + 1) & ~1);               // uint16 x 4 mi
    L.sblkc = L.sinfo + 2 * (max_blk + dpmax);         // int4 per slot
    L.total = L.sblkc + 8 * max_blk;
    return L;
}

template <int TAU>
__global__ void __launch_bounds__(kTanThreads, TAN5_MINB) tangent_row5_kernel(TangentArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int N = a.N;
    const int4 d0 = __ldg(a.rowdesc + 2 * blockIdx.x), d1 = __ldg(a.rowdesc + 2 * blockIdx.x + 1);
    const int A = d0.x, i0 = d0.y, ninc = d0.z, k0 = d0.w;
    const int nblk = d1.x, cb = d1.y, kdiag = d1.z;
    const int NT = a.NT, n0 = blockIdx.y * NT, nt = min(NT, N - n0);
    const Tan5Smem Ls = tan5_layout(a.max_inc, a.max_blk, NT);
    double* summ = sm + Ls.summ;   // [i][8][t]
    double* su = sm + Ls.su;       // [j][c][t]; later [part][8][t] diagonal partials
    double* incg = sm + Ls.incg;   // [i][24]
    double* rec = sm + Ls.rec;     // [p][8]
    uint16_t* scont = reinterpret_cast<uint16_t*>(sm + Ls.scont);
    int4* sinfo = reinterpret_cast<int4*>(sm + Ls.sinfo);  // per slot {c0, c1, j, bfix}
    double* sblkc = sm + Ls.sblkc;                          // [j][8]
    const int dparts = (ninc + kTanPart - 1) / kTanPart;    // the diagonal has one contribution per incidence
    const int nslots = dparts + nblk - 1;
    const bool afix = __ldg(a.dir + A) != 0;
    const double rho = a.rho, diffc = 3.0 * a.nu * a.nu, dAB = kQA - kQB;

    // ---- stage A
    // neighbour velocities: warp per block, lanes over its 3 x nt samples
    {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int j = wid; j < nblk; j += nw) {
            const double* src = a.state + (long)__ldg(a.col_idx + k0 + j) * 4 * N + n0;
            double* dst = su + j * 3 * NT;
            if (nt == N) {
                for (int e = lane; e < 3 * N; e += 32)
                    dst[e] = __ldg(src + e);
            } else {
                for (int e = lane; e < 3 * nt; e += 32) {
                    const int c = e / nt, t = e - c * nt;
                    dst[c * NT + t] = __ldg(src + c * N + t);
                }
            }
        }
    }
    for (int i = threadIdx.x; i < ninc; i += blockDim.x) {
        const int4 r1 = __ldg(a.inc_rec + 2 * (i0 + i) + 1);
        const int e = r1.x & 0x3FFFFFFF, la = (unsigned)r1.x >> 30;
        const double2* g = reinterpret_cast<const double2*>(a.tgeom + (long)kTGeo * e);
        double2* o = reinterpret_cast<double2*>(incg + i * kIncg);
        double2 v[10];
#pragma unroll
        for (int k = 0; k < 10; ++k)
            v[k] = __ldg(g + k);
        // gradN 0..11 | V 12 | xi00 2xi01 2xi02 xi11 2xi12 xi22 13..18 | diff 19 | meta 20
#pragma unroll
        for (int k = 0; k < 6; ++k)
            o[k] = v[k];
        o[6] = make_double2(v[6].x, v[6].y);                      // V, xi00
        o[7] = make_double2(2.0 * v[7].x, 2.0 * v[7].y);          // 2xi01, 2xi02
        o[8] = make_double2(v[8].x, 2.0 * v[8].y);                // xi11, 2xi12
        o[9] = make_double2(v[9].x, diffc * v[9].y);              // xi22, diff
        o[10] = make_double2(__longlong_as_double((long long)la | ((long long)(unsigned)r1.y << 8)), 0.0);
    }
    for (int p = threadIdx.x; p < 4 * ninc; p += blockDim.x)
        scont[p] = a.contrib[cb + p];
    for (int s = threadIdx.x; s < nslots; s += blockDim.x) {
        int4 info;
        if (s < dparts) {
            const int dc0 = __ldg(a.contrib_ptr + k0 + kdiag) - cb;
            info.x = dc0 + s * kTanPart;
            info.y = min(info.x + kTanPart, dc0 + ninc);
            info.z = kdiag;
            info.w = afix;
        } else {
            const int j = a.blk_order[k0 + s - dparts];
            info.x = __ldg(a.contrib_ptr + k0 + j) - cb;
            info.y = __ldg(a.contrib_ptr + k0 + j + 1) - cb;
            info.z = j;
            info.w = __ldg(a.dir + __ldg(a.col_idx + k0 + j)) != 0;
        }
        sinfo[s] = info;
    }
    for (int it = threadIdx.x; it < nblk * 4; it += blockDim.x)
        reinterpret_cast<double2*>(sblkc)[it] = __ldg(reinterpret_cast<const double2*>(a.blkc) + (long)k0 * 4 + it);
    __syncthreads();

    // ---- contribution records (list order) and phase 1 summaries
    for (int p = threadIdx.x; p < 4 * ninc; p += blockDim.x) {
        const int ent = scont[p];
        const int i = ent >> 2, b = ent & 3;
        const double* gi = incg + i * kIncg;
        const int la = int((unsigned long long)__double_as_longlong(gi[20]) & 3u);
        const double ga0 = gi[3 * la], ga1 = gi[3 * la + 1], ga2 = gi[3 * la + 2];
        const double gb0 = gi[3 * b], gb1 = gi[3 * b + 1], gb2 = gi[3 * b + 2];
        double2* o = reinterpret_cast<double2*>(rec + p * 8);
        o[0] = make_double2(ga0, ga1);
        o[1] = make_double2(ga2, fma(ga0, gb0, fma(ga1, gb1, ga2 * gb2)));
        o[2] = make_double2(gb0, gb1);
        o[3] = make_double2(gb2, __longlong_as_double((long long)i * 8 * NT));
    }
    const int di = blockDim.x / nt, dt = blockDim.x - di * nt;
    const int i_start = threadIdx.x / nt, t_start = threadIdx.x - i_start * nt;
    for (int it = threadIdx.x, i = i_start, t = t_start; it < ninc * nt;
             it += blockDim.x, t += dt, i += di + (t >= nt), t -= (t >= nt ? nt : 0)) {
        const double* gi = incg + i * kIncg;
        const double2 xv = *reinterpret_cast<const double2*>(gi + 12);  // V, xi00
        const double2 x1 = *reinterpret_cast<const double2*>(gi + 14);  // 2xi01, 2xi02
        const double2 x2 = *reinterpret_cast<const double2*>(gi + 16);  // xi11, 2xi12
        const double2 x3 = *reinterpret_cast<const double2*>(gi + 18);  // xi22, diff
        const unsigned long long meta = (unsigned long long)__double_as_longlong(gi[20]);
        const int la = int(meta & 3u);
        const unsigned cols = unsigned(meta >> 8);
        const double ga[3] = {gi[3 * la], gi[3 * la + 1], gi[3 * la + 2]};
        const double V = xv.x, w = 0.25 * V;
        auto quad = [&](const double v[3]) {
            const double r0 = fma(x1.y, v[2], fma(x1.x, v[1], xv.y * v[0]));
            const double r1 = fma(x2.y, v[2], x2.x * v[1]);
            return fma(v[0], r0, fma(v[1], r1, fma(v[2], x3.x * v[2], x3.y)));
        };
        double u[4][3], usum[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double* sb = su + (size_t)((cols >> (8 * b)) & 0xFFu) * 3 * NT + t;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                u[b][c] = sb[c * NT];
                usum[c] += u[b][c];
            }
        }
        double bu[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            bu[c] = kQB * usum[c];
        bool bad = false;
        double tau_mean = 0.0;
        if (TAU == 1) {
            const double um[3] = {0.25 * usum[0], 0.25 * usum[1], 0.25 * usum[2]};
            const double arg = quad(um);
            bad = !(arg > 0.0);
            tau_mean = tau_or_zero(arg, bad);
        }
        double asum = 0.0, tsum = 0.0, z[3] = {0.0, 0.0, 0.0}, kap[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double uq[3];
#pragma unroll
            for (int c = 0; c < 3; ++c)
                uq[c] = fma(dAB, u[q][c], bu[c]);
            double tq = tau_mean;
            if (TAU == 0) {
                const double arg = quad(uq);
                const bool bq = !(arg > 0.0);
                bad |= bq;
                tq = tau_or_zero(arg, bq);
            }
            const double tadv = tq * fma(uq[0], ga[0], fma(uq[1], ga[1], uq[2] * ga[2]));
            const double na = (q == la) ? kQA : kQB;
            asum += tadv;
            tsum += tq;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                z[c] = fma(tq, uq[c], z[c]);
                kap[c] = fma(na + tadv, uq[c], kap[c]);
            }
        }
        if (bad)
            atomicOr(a.flag, 1);
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

    // ---- phase 2: per (slot, sample) register accumulation
    double* dpart = su;
    const double mu = a.mu, pc = a.pseudo_c;
    for (int it = threadIdx.x, slot = i_start, t = t_start; it < nslots * nt;
             it += blockDim.x, t += dt, slot += di + (t >= nt), t -= (t >= nt ? nt : 0)) {
        const int n = n0 + t;
        const int4 info = sinfo[slot];
        const int j = info.z;
        const bool bfix = info.w != 0;
        double K = 0.0, G0 = 0.0, G1 = 0.0, G2 = 0.0, D0 = 0.0, D1 = 0.0, D2 = 0.0, L = 0.0;
#pragma unroll 2
        for (int p = info.x; p < info.y; ++p) {
            const double2* r = reinterpret_cast<const double2*>(rec + p * 8);
            const double2 ra = r[0], rb = r[1], rc = r[2], rd = r[3];
            const double* s = summ + __double_as_longlong(rd.y) + t;
            const double gb0 = rc.x, gb1 = rc.y, gb2 = rd.x;
            K = fma(s[0], gb0, fma(s[NT], gb1, fma(s[2 * NT], gb2, K)));
            const double al = s[3 * NT];
            G0 = fma(al, gb0, G0);
            G1 = fma(al, gb1, G1);
            G2 = fma(al, gb2, G2);
            const double alb = fma(s[4 * NT], gb0, fma(s[5 * NT], gb1, s[6 * NT] * gb2));
            D0 = fma(ra.x, alb, D0);
            D1 = fma(ra.y, alb, D1);
            D2 = fma(rb.x, alb, D2);
            L = fma(rb.y, s[7 * NT], L);
        }
        if (slot >= dparts || slot == 0) {
            const double2* bc = reinterpret_cast<const double2*>(sblkc + j * 8);
            const double2 b0 = bc[0], b1 = bc[1], b2 = bc[2], b3 = bc[3];
            K += fma(mu, b0.x, pc * b0.y);
            G0 += b1.x;
            G1 += b1.y;
            G2 += b2.x;
            D0 += b2.y;
            D1 += b3.x;
            D2 += b3.y;
        }
        if (afix || bfix)
            K = 0.0;
        if (afix)
            G0 = G1 = G2 = 0.0;
        if (bfix)
            D0 = D1 = D2 = 0.0;
        if (slot >= dparts) {
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
            double* o = dpart + (size_t)slot * 8 * NT + t;
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

// Per block: the n-invariant sums of the v5 update in element order (setup,
// geometry only): {sum V gg, sum V m_ab, sum -w dN_a (3), sum w dN_b (3)}.
__global__ void tangent_blockconst_kernel(const double* __restrict__ tgeom,
                                          const int* __restrict__ row_ptr,
                                          const int* __restrict__ inc_ptr,
                                          const int4* __restrict__ inc_rec,
                                          const int* __restrict__ contrib_ptr,
                                          const uint16_t* __restrict__ contrib, int nn,
                                          double* __restrict__ blkc) {
    const int A = blockIdx.x * blockDim.x + threadIdx.x;
    if (A >= nn)
        return;
    const int i0 = inc_ptr[A];
    for (int k = row_ptr[A]; k < row_ptr[A + 1]; ++k) {
        double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int p = contrib_ptr[k]; p < contrib_ptr[k + 1]; ++p) {
            const int i = contrib[p] >> 2, b = contrib[p] & 3;
            const int4 r1 = inc_rec[2 * (i0 + i) + 1];
            const int e = r1.x & 0x3FFFFFFF, la = (unsigned)r1.x >> 30;
            const double* g = tgeom + (long)kTGeo * e;
            const double V = g[12], w = 0.25 * V;
            const double gg = g[3 * la] * g[3 * b] + g[3 * la + 1] * g[3 * b + 1] +
                              g[3 * la + 2] * g[3 * b + 2];
            s[0] += V * gg;
            s[1] += V * (b == la ? 0.1 : 0.05);
            for (int c = 0; c < 3; ++c) {
                s[2 + c] -= w * g[3 * la + c];
                s[5 + c] += w * g[3 * b + c];
            }
        }
        for (int c = 0; c < 8; ++c)
            blkc[(long)k * 8 + c] = s[c];
    }
}

void launch_tangent_blockconst(const double* tgeom, const int* row_ptr, const int* inc_ptr,
                               const int4* inc_rec, const int* contrib_ptr, const uint16_t* contrib,
                               int nn, double* blkc, cudaStream_t st) {
    if (nn <= 0)
        return;
    note_launch();
    tangent_blockconst_kernel<<<(nn + 127) / 128, 128, 0, st>>>(tgeom, row_ptr, inc_ptr, inc_rec,
                                                               contrib_ptr, contrib, nn, blkc);
}

size_t tangent_row_smem(int max_inc, int max_blk, int max_dparts, int NT) {
    (void)max_dparts;
    return sizeof(double) * (size_t)tan5_layout(max_inc, max_blk, NT).total;
}

cudaError_t configure_tangent_row_smem(size_t bytes) {
    const int b = int(bytes < 48 * 1024 ? 48 * 1024 : bytes);
    cudaError_t e = cudaFuncSetAttribute(tangent_row5_kernel<0>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e != cudaSuccess)
        return e;
    return cudaFuncSetAttribute(tangent_row5_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

void launch_tangent_row(const TangentArgs& a, int nrows, size_t smem, cudaStream_t st) {
    if (nrows <= 0)
        return;
    note_launch();
    const dim3 grid(nrows, (a.N + a.NT - 1) / a.NT);
    if (a.tau_mode == 1)
        tangent_row5_kernel<1><<<grid, kTanThreads, smem, st>>>(a);
    else
        tangent_row5_kernel<0><<<grid, kTanThreads, smem, st>>>(a);
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
