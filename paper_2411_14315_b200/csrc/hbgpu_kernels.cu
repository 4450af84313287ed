// CUDA kernels of the B200-native HB-GLS hot path (sm_100a, FP64).
//
// Reference (CPU C++, /root/reference/proj) loops being replaced:
//   element_residual + scatter   src/assembly.cpp:141-263, 465-521
//   nodal H passes               src/assembly.cpp:453-463, 523-535 (FFTW there, dense N x N here)
//   boundary terms               src/assembly.cpp:376-413
//   element_tangent_p + scatter  src/assembly.cpp:265-374, 550-666
//   assemble_mass                src/assembly.cpp:668-681
//   TangentOperator::matvec      src/linalg.cpp:41-128
//   jacobi_preconditioner        src/linalg.cpp:130-154
//   gmres_solve vector work      src/linalg.cpp:167-293
//
// Every kernel is deterministic: no floating-point atomics, fixed reduction
// trees, fixed summation order per output (element order for the tangent /
// mass, (chunk, element, local index) order for the residual).
#include "hbgpu_internal.h"

#include <cstring>

namespace hbgpu {

std::atomic<long long> g_launches{0};

namespace {
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace

// ---------------------------------------------------------------- geometry

// element_geometry (mesh.cpp:159-203), one thread per element.
__global__ void geometry_kernel(const double* __restrict__ xyz, const int4* __restrict__ conn,
                                int ne, double* __restrict__ geom, int* flag) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne)
        return;
    const int4 c = conn[e];
    const int nd[4] = {c.x, c.y, c.z, c.w};
    double x[4][3];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            x[a][i] = xyz[3 * (long)nd[a] + i];
    double c0[3], c1[3], c2[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        c0[i] = x[1][i] - x[0][i];
        c1[i] = x[2][i] - x[0][i];
        c2[i] = x[3][i] - x[0][i];
    }
    const double det = c0[0] * (c1[1] * c2[2] - c1[2] * c2[1]) -
                       c1[0] * (c0[1] * c2[2] - c0[2] * c2[1]) +
                       c2[0] * (c0[1] * c1[2] - c0[2] * c1[1]);
    double* g = geom + 22 * (long)e;
    g[12] = det / 6.0;
    if (!(det / 6.0 > 0.0))
        atomicOr(flag, 2);
    const double r0[3] = {c1[1] * c2[2] - c1[2] * c2[1], c1[2] * c2[0] - c1[0] * c2[2],
                          c1[0] * c2[1] - c1[1] * c2[0]};
    const double r1[3] = {c2[1] * c0[2] - c2[2] * c0[1], c2[2] * c0[0] - c2[0] * c0[2],
                          c2[0] * c0[1] - c2[1] * c0[0]};
    const double r2[3] = {c0[1] * c1[2] - c0[2] * c1[1], c0[2] * c1[0] - c0[0] * c1[2],
                          c0[0] * c1[1] - c0[1] * c1[0]};
    double j[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        j[0][i] = r0[i] / det;
        j[1][i] = r1[i] / det;
        j[2][i] = r2[i] / det;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        g[3 * 1 + i] = j[0][i];
        g[3 * 2 + i] = j[1][i];
        g[3 * 3 + i] = j[2][i];
        g[i] = -(j[0][i] + j[1][i] + j[2][i]);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            g[13 + 3 * a + b] = j[0][a] * j[0][b] + j[1][a] * j[1][b] + j[2][a] * j[2][b];
}

void launch_geometry(const double* xyz, const int4* conn, int ne, double* geom, int* flag,
                     cudaStream_t st) {
    if (ne <= 0)
        return;
    note_launch();
    geometry_kernel<<<(ne + 255) / 256, 256, 0, st>>>(xyz, conn, ne, geom, flag);
}

// ---------------------------------------------------------------- nodal H

// out[(A*os + i*N) + n] = sum_m H[n][m] in[(A*is + i*N) + m], i < 3: the
// batched pseudo-spectral derivative of every velocity series
// (assembly.cpp:453-463; SpectralOperators::apply_many, spectral.cpp:185-227).
// It is a small GEMM, OUT[3 nn x N] = X[3 nn x N] H^T[N x N], run on the FP64
// tensor cores (mma.sync.m8n8k4.f64, SASS DMMA): a warp owns 8-series x
// 8-sample output tiles and walks m in steps of 4 (two shared loads per
// 256-FMA instruction); N is zero-padded to a multiple of 8.  A CTA takes 32
// nodes (96 series).  On B200 the DMMA and DFMA paths share one FP64
// throughput (tools/fp64_probe.cu: 37.2 / 37.1 TFLOP/s alone, 35.3 together),
// so DMMA wins only where a DFMA formulation is bound by its shared-memory
// operand traffic — as the register-tiled DFMA version of this pass was
// (4 series x SPT samples per thread, 7 shared loads per 12 FMA): config 4
// (N = 47) 0.864 -> 0.787 ms, config 1 (N = 19) 0.039 -> 0.030 ms with DMMA;
// the round-1 per-(series, sample) dot product took 2.53 ms at config 4.
constexpr int kHmNodes = 32, kHmSeries = 3 * kHmNodes, kHmThreads = 256;
__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(kHmThreads) apply_h_dmma_kernel(const double* __restrict__ H, int N,
                                                                  const double* __restrict__ in, int is,
                                                                  double* __restrict__ out, int os, int nnodes) {
    extern __shared__ double sh[];
    const int NP = (N + 7) & ~7, LS = NP + 4;  // padded sample count, smem row stride
    double* Ht = sh;                           // [m][LS]: Ht[m][n] = H[n][m], zero-padded
    double* Xs = sh + NP * LS;                 // [series][LS], zero-padded in m
    for (int k = threadIdx.x; k < NP * NP; k += blockDim.x) {
        const int m = k / NP, n = k - m * NP;
        Ht[m * LS + n] = (m < N && n < N) ? H[n * N + m] : 0.0;
    }
    const long A0 = (long)blockIdx.x * kHmNodes;
    const int nloc = (int)min((long)kHmNodes, (long)nnodes - A0);
    for (int k = threadIdx.x; k < kHmSeries * NP; k += blockDim.x) {
        const int sl = k / NP, m = k - sl * NP, ln = sl / 3, i = sl - 3 * ln;
        Xs[sl * LS + m] = (ln < nloc && m < N) ? __ldg(in + (A0 + ln) * is + (long)i * N + m) : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = lane >> 2, q = lane & 3;
    const int ntn = NP / 8, tiles = (kHmSeries / 8) * ntn;
    for (int tile = warp; tile < tiles; tile += kHmThreads / 32) {
        const int ts = tile / ntn, tn = tile - ts * ntn;
        const double* xa = Xs + (ts * 8 + r) * LS + q;  // A[r][k] = X[s0 + r][k0 + q]
        const double* hb = Ht + q * LS + tn * 8 + r;     // B[k][n] = Ht[k0 + q][n0 + r]
        double c0 = 0.0, c1 = 0.0;
        for (int k0 = 0; k0 < NP; k0 += 4)
            dmma_m8n8k4(c0, c1, xa[k0], hb[k0 * LS]);
        const int sl = ts * 8 + r, ln = sl / 3, i = sl - 3 * ln;
        if (ln < nloc) {
            double* o = out + (A0 + ln) * os + (long)i * N;
            const int n = tn * 8 + 2 * q;
            if (n < N)
                o[n] = c0;
            if (n + 1 < N)
                o[n + 1] = c1;
        }
    }
}

void launch_apply_h_series(const double* H, int N, const double* in, int in_node_stride,
                           double* out, int out_node_stride, int nnodes, cudaStream_t st) {
    if (nnodes <= 0)
        return;
    const int NP = (N + 7) & ~7, LS = NP + 4;
    const size_t smem = sizeof(double) * ((size_t)NP * LS + (size_t)kHmSeries * LS);
    static bool configured = false;  // N up to 63: ~87 KB (above the 48 KB default)
    if (!configured) {
        cudaFuncSetAttribute(apply_h_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        configured = true;
    }
    note_launch();
    apply_h_dmma_kernel<<<(nnodes + kHmNodes - 1) / kHmNodes, kHmThreads, smem, st>>>(
        H, N, in, in_node_stride, out, out_node_stride, nnodes);
}

// ---------------------------------------------------------------- residual


// Element residual at one (element, sample) with the quadrature sums
// factored (W-trick), reading nodal data from shared memory and writing the
// 28 element outputs into the element's shared-memory slots:
//   r_m[a][i] = mu V gradN_a.grad u_i - dN_a/dx_i (V/4) sum p + rho V/20 (sum_b Hu_b,i + Hu_a,i)
//             + w rho (B Cs_i + (A-B) conv_{q=a,i}) + w gradN_a . W_{:,i}
//   s[a][i]   = w (B TLs_i + (A-B) tl_{q=a,i})
//   r_c[a]    = w div u + (w/rho) gradN_a . TLs
// with conv_q = u_q . grad u, tl_q = tau_q (rho Hu_q + rho conv_q + grad p),
// Cs = sum_q conv_q, TLs = sum_q tl_q, W_ji = sum_q u_q,j tl_q,i.  Algebraically
// identical to element_residual (assembly.cpp:141-263): N_a(q) = B + (A-B) delta_aq.
// Slot layout: out[(a*7 + c) * T], c = 0..2 r_m, 3 r_c, 4..6 s.
// Shared-memory operand read the compiler may not hoist or keep live: the
// element kernels re-read geometry / nodal operands where they are used
// instead of pinning ~50 doubles in registers (which forced spills).
__device__ __forceinline__ double lds(const double* p) {
    double v;
#if RES_VOLATILE_LDS
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
#else
    v = *p;
#endif
    return v;
}
struct SmemRow {
    const double* p;
    __device__ __forceinline__ double operator[](int k) const { return lds(p + k); }
};

__device__ __forceinline__ void element_residual_smem(const double* __restrict__ gsm,
                                                      const double* __restrict__ nd, int ndst,
                                                      const int lc[4], int T, int t,
                                                      double rho, double inv_rho, double mu, double nu,
                                                      int tau_mode, int* flag,
                                                      double* __restrict__ out) {
    // nd: node data [ln][c][t], c = u0 u1 u2 p hu0 hu1 hu2, node stride ndst
    const SmemRow g{gsm};
    auto U = [&](int b, int c) { return lds(nd + lc[b] * ndst + c * T + t); };
    const double V = g[12], w = 0.25 * V;
    double gu[3][3], gp[3], usum[3], hsum[3], psum = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        gp[i] = 0.0;
        usum[i] = 0.0;
        hsum[i] = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
            gu[i][j] = 0.0;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const double pb = U(b, 3);
        psum += pb;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double ub = U(b, i);
            usum[i] += ub;
            hsum[i] += U(b, 4 + i);
            gp[i] += g[3 * b + i] * pb;
#pragma unroll
            for (int j = 0; j < 3; ++j)
                gu[i][j] += g[3 * b + j] * ub;
        }
    }
    const double div = gu[0][0] + gu[1][1] + gu[2][2];
    // compact geometry record (tangent_geometry_kernel): xi00 xi01 xi02 xi11 xi12 xi22 at
    // 13..18, xi:xi at 19; u . xi . u in symmetric form
    const double diff = 3.0 * nu * nu * g[19];
    auto quad = [&](const double v[3]) {
        const double q0 = fma(2.0 * g[15], v[2], fma(2.0 * g[14], v[1], g[13] * v[0]));
        const double q1 = fma(2.0 * g[17], v[2], g[16] * v[1]);
        return fma(v[0], q0, fma(v[1], q1, fma(v[2], g[18] * v[2], diff)));
    };
    bool bad = false;
    double tau_mean = 0.0;
    if (tau_mode == 1) {
        const double um[3] = {0.25 * usum[0], 0.25 * usum[1], 0.25 * usum[2]};
        const double arg = quad(um);
        bad = !(arg > 0.0);
        tau_mean = tau_or_zero(arg, bad);
    }
    const double dAB = kQA - kQB;
    double Cs[3] = {0, 0, 0}, TLs[3] = {0, 0, 0}, W[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    double tauq[4];
    // pass 1 over the quadrature points: the q-sums Cs, TLs, W (and tau_q)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double uq[3], huq[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            uq[i] = kQB * usum[i] + dAB * U(q, i);
            huq[i] = kQB * hsum[i] + dAB * U(q, 4 + i);
        }
        double tau = tau_mean;
        if (tau_mode == 0) {
            const double arg = quad(uq);
            const bool bq = !(arg > 0.0);
            bad |= bq;
            tau = tau_or_zero(arg, bq);
        }
        tauq[q] = tau;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double cv = uq[0] * gu[i][0] + uq[1] * gu[i][1] + uq[2] * gu[i][2];
            const double tl = tau * (rho * huq[i] + rho * cv + gp[i]);
            Cs[i] += cv;
            TLs[i] += tl;
#pragma unroll
            for (int j = 0; j < 3; ++j)
                W[j][i] += uq[j] * tl;
        }
    }
    if (bad)
        atomicOr(flag, 1);
    // pass 2, node a = quadrature point a: the q = a parts (conv_q, tl_q
    // recomputed from tau_a) plus the q-sum and Galerkin terms, each output
    // written once
    // rho V / 20 and w / rho as multiplications (two FP64 divisions per (element, sample) otherwise)
    const double muV = mu * V, moff = rho * V * 0.05, wr = w * inv_rho;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const double ga0 = g[3 * a], ga1 = g[3 * a + 1], ga2 = g[3 * a + 2];
        double uq[3], huq[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            uq[i] = kQB * usum[i] + dAB * U(a, i);
            huq[i] = U(a, 4 + i);  // raw nodal Hu_a (Galerkin mass term), huq at q = a below
        }
        double* oa = out + a * 7 * T;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double cv = uq[0] * gu[i][0] + uq[1] * gu[i][1] + uq[2] * gu[i][2];
            const double hq = kQB * hsum[i] + dAB * huq[i];
            const double tl = tauq[a] * (rho * hq + rho * cv + gp[i]);
            const double gai = g[3 * a + i];
            oa[i * T] = w * rho * dAB * cv +
                        (muV * (ga0 * gu[i][0] + ga1 * gu[i][1] + ga2 * gu[i][2]) - gai * w * psum +
                         moff * (hsum[i] + huq[i]) + w * rho * kQB * Cs[i] +
                         w * (ga0 * W[0][i] + ga1 * W[1][i] + ga2 * W[2][i]));
            oa[(4 + i) * T] = w * dAB * tl + w * kQB * TLs[i];
        }
        oa[3 * T] = w * div + wr * (ga0 * TLs[0] + ga1 * TLs[1] + ga2 * TLs[2]);
    }
}

// Residual element pass as a persistent pipeline.  CTA b walks element
// chunks b, b+G, ... and, per chunk, its time-sample tiles (T samples, residual_tile(N)).
//  * The chunk's metadata ("chunk pack": local nodes, per-node slot lists,
//    local connectivity) and its 64 geometry records arrive by bulk async copy
//    (cp.async.bulk on an mbarrier), issued one chunk ahead.
//  * The nodal data (u, p, Hu) of the next tile is gathered with cp.async
//    (LDGSTS) while the current tile computes: one thread per (chunk node,
//    component) issues the tile's samples, addresses come from shared memory.
//  * Per tile: one (element, sample) per thread into per-element slots, then
//    every chunk node's slots are reduced in fixed (element, local index)
//    order and written as one partial record.  Partials are tile-major and
//    contiguous per chunk: partial[((tile*npairs + p)*7 + c)*T + t].
// Deterministic, no atomics.
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(K));
}

__host__ __device__ inline int rp_align16(int bytes) { return (bytes + 15) & ~15; }
struct ResPackSec {
    int nodes, sptr, soff, lconn, total;
};
__host__ __device__ inline ResPackSec res_pack_sections(int nloc, int ecount) {
    ResPackSec s;
    s.nodes = 16;
    s.sptr = s.nodes + rp_align16(4 * nloc);
    s.soff = s.sptr + rp_align16(4 * (nloc + 1));
    s.lconn = s.soff + rp_align16(2 * 4 * ecount);
    s.total = s.lconn + rp_align16(4 * ecount);
    return s;
}
size_t residual_pack_bytes(int nloc, int ecount) { return (size_t)res_pack_sections(nloc, ecount).total; }

void residual_pack_write(unsigned char* dst, int nloc, int ecount, int nb, const int* nodes,
                         const int* sptr_rel, const uint16_t* soff, const uint32_t* lconn) {
    const ResPackSec s = res_pack_sections(nloc, ecount);
    memset(dst, 0, (size_t)s.total);
    int* h = reinterpret_cast<int*>(dst);
    h[0] = nloc;
    h[1] = ecount;
    h[2] = nb;
    memcpy(dst + s.nodes, nodes, sizeof(int) * (size_t)nloc);
    memcpy(dst + s.sptr, sptr_rel, sizeof(int) * (size_t)(nloc + 1));
    memcpy(dst + s.soff, soff, sizeof(uint16_t) * (size_t)(4 * ecount));
    memcpy(dst + s.lconn, lconn, sizeof(uint32_t) * (size_t)ecount);
}

// shared-memory node-record stride of the residual tiles: 7T doubles, unpadded.  A
// warp's nodal load is eight 32-byte runs (8 elements x 4 samples); with the stride
// 28 doubles = 24 words (mod 32) every run starts on an 8-bank boundary, so two runs
// either coincide in their banks or do not touch (25% of node pairs conflict).  The
// round-1 pad to 7T + 1 put consecutive nodes 6 banks apart, where 44% of the pairs
// overlap partially: config 4 element pass 22.24 -> 21.60 ms without it
// (profiles/r2w_kbench.log; ncu r2p: 4.13 wavefronts per nodal load against 2 ideal).
#ifndef RES_GATHER_LINEAR
#define RES_GATHER_LINEAR 2
#endif
#ifndef RES_ND_PAD
#define RES_ND_PAD 0
#endif
__host__ __device__ constexpr int res_nd_stride(int T) { return 7 * T + ((T == 4 && RES_ND_PAD) ? 1 : 0); }

struct ResSmem {
    int pk, geo, nd, slots, mbar, total;  // byte offsets
};
__host__ __device__ inline ResSmem res_layout(int max_nloc, int max_rpack, int T) {
    constexpr int CE = kChunkElems;
    ResSmem L;
    L.pk = 0;                                              // 2 x max_rpack
    L.geo = L.pk + 2 * rp_align16(max_rpack);              // 2 x [CE][kTGeo]
    L.nd = L.geo + 2 * CE * kTGeo * 8;                     // 2 x [nloc][7][T]
    L.slots = L.nd + 2 * max_nloc * res_nd_stride(T) * 8;  // [CE][29T]
    L.mbar = L.slots + CE * 29 * T * 8;
    L.total = L.mbar + 16;
    return L;
}
size_t residual_smem_bytes(int max_nloc, int max_rpack, int T) {
    return (size_t)res_layout(max_nloc, max_rpack, T).total;
}

// T = time samples per tile (4; 1 when N is small, where a 4-sample tile would
// leave most threads idle — the host picks it, residual_tile()).
template <int T>
__global__ void __launch_bounds__(kChunkElems * T, RES_MINB * 4 / T) residual_chunk_kernel(ResidualChunkArgs a) {
    extern __shared__ __align__(128) unsigned char smraw[];
    constexpr int CE = kChunkElems, ndst = 7 * T, es = 29 * T, nds = res_nd_stride(T);
    const int N = a.N, nch = a.nchunks;
    const int ntiles = (N + T - 1) / T;
    const ResSmem Ls = res_layout(a.max_nloc, a.max_rpack, T);
    const int mpk = rp_align16(a.max_rpack);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smraw + Ls.mbar);
    double* slots = reinterpret_cast<double*>(smraw + Ls.slots);
    int ch = blockIdx.x;
    if (ch >= nch)
        return;
    const double inv_rho = 1.0 / a.rho;
    if (threadIdx.x == 0) {
        mbar_init(mbar, 1);
        mbar_init(mbar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue_pack = [&](int c, int slot) {  // one thread
        const int p0 = __ldg(a.rpack_ptr + c), p1 = __ldg(a.rpack_ptr + c + 1);
        const int ecount = min(CE, a.ne - c * CE);
        const uint32_t pb = (uint32_t)(p1 - p0) * 16u, gb = (uint32_t)ecount * kTGeo * 8u;
        mbar_expect_tx(mbar + slot, pb + gb);
        bulk_g2s(smraw + Ls.pk + slot * mpk, a.rpack + (size_t)p0 * 16, pb, mbar + slot);
        bulk_g2s(smraw + Ls.geo + slot * CE * kTGeo * 8, a.tgeom + (size_t)c * CE * kTGeo, gb, mbar + slot);
    };
    auto issue_tile = [&](int slot, int tile, int b) {  // all threads
        const unsigned char* pk = smraw + Ls.pk + slot * mpk;
        const int* h = reinterpret_cast<const int*>(pk);
        const int nloc = h[0];
        const ResPackSec s = res_pack_sections(nloc, h[1]);
        const int* nodes = reinterpret_cast<const int*>(pk + s.nodes);
        double* nd = reinterpret_cast<double*>(smraw + Ls.nd) + (size_t)b * a.max_nloc * nds;
        const int n0 = tile * T;
#if RES_GATHER_LINEAR == 2
        // thread per (node, component, sample pair): stores 16 B apart
        constexpr int P = (T % 2 == 0) ? 2 : 1, TG = T / P;
        for (int k = threadIdx.x; k < nloc * 7 * TG; k += blockDim.x) {
            const int ln = k / (7 * TG), rem = k - ln * 7 * TG, cc = rem / TG, t = P * (rem - cc * TG);
            // 32-bit element offsets (4 nn N < 2^32 is checked in hbgpu_set_basis)
            const unsigned A = (unsigned)nodes[ln];
            const double* src = cc < 4 ? a.state + ((A * 4u + (unsigned)cc) * (unsigned)N + (unsigned)n0)
                                       : a.hu + ((A * 3u + (unsigned)(cc - 4)) * (unsigned)N + (unsigned)n0);
            double* dst = nd + ln * nds + cc * T + t;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                if (n0 + t + q < N)
                    cp_async8(dst + q, src + t + q);
                else
                    dst[q] = 0.0;
            }
        }
#elif RES_GATHER_LINEAR
        // thread per (node, component, sample), sample fastest: a warp's shared
        // stores are one contiguous run (the per-(node, component) mapping put
        // consecutive threads 4 doubles apart: 8-way bank conflicts)
        for (int k = threadIdx.x; k < nloc * 7 * T; k += blockDim.x) {
            const int ln = k / (7 * T), rem = k - ln * 7 * T, cc = rem / T, t = rem - cc * T;
            const long A = nodes[ln];
            const double* src = cc < 4 ? a.state + (A * 4 + cc) * N + n0 : a.hu + (A * 3 + (cc - 4)) * N + n0;
            double* dst = nd + ln * nds + rem;
            if (n0 + t < N)
                cp_async8(dst, src + t);
            else
                *dst = 0.0;
        }
#else
        for (int k = threadIdx.x; k < nloc * 7; k += blockDim.x) {
            const int ln = k / 7, cc = k - 7 * ln;
            const long A = nodes[ln];
            const double* src = cc < 4 ? a.state + (A * 4 + cc) * N + n0 : a.hu + (A * 3 + (cc - 4)) * N + n0;
            double* dst = nd + ln * nds + cc * T;
#pragma unroll
            for (int t = 0; t < T; ++t) {
                if (n0 + t < N)
                    cp_async8(dst + t, src + t);
                else
                    dst[t] = 0.0;
            }
        }
#endif
    };

    if (threadIdx.x == 0)
        issue_pack(ch, 0);
    mbar_wait(mbar, 0);
    issue_tile(0, 0, 0);
    cp_async_commit();
    int gt = 0;
    for (int jj = 0; ch < nch; ++jj, ch += gridDim.x) {
        const int ps = jj & 1, nextch = ch + gridDim.x;
        const unsigned char* pk = smraw + Ls.pk + ps * mpk;
        const int* h = reinterpret_cast<const int*>(pk);
        const int nloc = h[0], ecount = h[1], nb = h[2];
        const ResPackSec sec = res_pack_sections(nloc, ecount);
        const int* sptr = reinterpret_cast<const int*>(pk + sec.sptr);
        const uint16_t* soff = reinterpret_cast<const uint16_t*>(pk + sec.soff);
        const uint32_t* lconn = reinterpret_cast<const uint32_t*>(pk + sec.lconn);
        const double* geo = reinterpret_cast<const double*>(smraw + Ls.geo + ps * CE * kTGeo * 8);
        for (int tile = 0; tile < ntiles; ++tile, ++gt) {
            const int b = gt & 1, n0 = tile * T;
            cp_async_wait<0>();
            __syncthreads();  // tile data visible; previous reduction done
            if (tile == 0 && threadIdx.x == 0 && nextch < nch)
                issue_pack(nextch, ps ^ 1);
            if (tile + 1 < ntiles) {
                issue_tile(ps, tile + 1, b ^ 1);
            } else if (nextch < nch) {
                mbar_wait(mbar + (ps ^ 1), ((jj + 1) >> 1) & 1);
                issue_tile(ps ^ 1, 0, b ^ 1);
            }
            cp_async_commit();
            const double* nd = reinterpret_cast<const double*>(smraw + Ls.nd) + (size_t)b * a.max_nloc * nds;
            {
                const int el = threadIdx.x / T, t = threadIdx.x - el * T;
                if (el < ecount && n0 + t < N) {
                    const uint32_t pkc = lconn[el];
                    const int lc[4] = {int(pkc & 0xFF), int((pkc >> 8) & 0xFF), int((pkc >> 16) & 0xFF),
                                       int(pkc >> 24)};
                    element_residual_smem(geo + el * kTGeo, nd, nds, lc, T, t, a.rho, inv_rho, a.mu, a.nu,
                                          a.tau_mode, a.flag, slots + el * es + t);
                }
            }
            __syncthreads();
            double* out = a.partial + ((long)tile * a.npairs + nb) * ndst;
            // thread per (chunk node, sample): walk the node's slot offsets once,
            // accumulating all 7 outputs.  This pass runs at the shared-memory wavefront
            // rate (ncu r2p: 94%); spreading it over more threads was slower both ways
            // tried at config 4: one thread per (node, output, sample), one 7x longer
            // dependent chain each, 22.2 -> 23.8 ms; two threads per (node, sample) with
            // 4 + 3 outputs 22.2 -> 23.8 ms (profiles/r2r_kbench.log, r2w_kbench.log)
            for (int k = threadIdx.x; k < nloc * T; k += blockDim.x) {
                const int ln = k / T, t = k - ln * T;
                double acc[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                const int q1 = sptr[ln + 1];
                for (int q = sptr[ln]; q < q1; ++q) {
                    const double* sp = slots + soff[q] * T + t;  // (el*29 + a*7) T
#pragma unroll
                    for (int cc = 0; cc < 7; ++cc)
                        acc[cc] += sp[cc * T];
                }
#pragma unroll
                for (int cc = 0; cc < 7; ++cc)
                    out[(ln * 7 + cc) * T + t] = acc[cc];
            }
        }
    }
    cp_async_wait<0>();
}

int residual_tile(int N) {
    // largest tile whose padding wastes at most 15% of the thread slots
    for (int T : {4, 2})
        if (N >= T && double(N) / double(((N + T - 1) / T) * T) >= 0.85)
            return T;
    return 1;
}

void launch_residual_chunks(const ResidualChunkArgs& a, int grid, int T, cudaStream_t st) {
    if (a.nchunks <= 0)
        return;
    note_launch();
    const size_t sm = residual_smem_bytes(a.max_nloc, a.max_rpack, T);
    const int g = min(grid, a.nchunks);
    if (T == 4)
        residual_chunk_kernel<4><<<g, kChunkElems * 4, sm, st>>>(a);
    else if (T == 2)
        residual_chunk_kernel<2><<<g, kChunkElems * 2, sm, st>>>(a);
    else
        residual_chunk_kernel<1><<<g, kChunkElems, sm, st>>>(a);
}

cudaError_t configure_residual_smem(size_t bytes, int T) {
    const int b = int(bytes < 48 * 1024 ? 48 * 1024 : bytes);
    if (T == 4)
        return cudaFuncSetAttribute(residual_chunk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (T == 2)
        return cudaFuncSetAttribute(residual_chunk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    return cudaFuncSetAttribute(residual_chunk_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

// Node pass: sums the node's chunk partials in chunk order, completes the
// least-squares rows r_u -= H s (assembly.cpp:523-535) and zeroes Dirichlet
// velocity rows (assembly.cpp:541-544).  Thread (node, n); the N threads of a
// node exchange s through shared memory for the dense H product.
__global__ void __launch_bounds__(256) residual_nodes_kernel(const double* __restrict__ H, int N,
                                                             int nn, int rows_per_cta,
                                                             const int* __restrict__ npart_ptr,
                                                             const int* __restrict__ npart,
                                                             const double* __restrict__ partial,
                                                             const uint8_t* __restrict__ dir,
                                                             double* __restrict__ r, int T,
                                                             long npairs) {
    extern __shared__ double sh[];
    double* sH = sh;
    double* ss = sh + N * N;
    for (int k = threadIdx.x; k < N * N; k += blockDim.x)
        sH[k] = H[k];
    const int rr = threadIdx.x / N, n = threadIdx.x - rr * N;
    const long A = (long)blockIdx.x * rows_per_cta + rr;
    const bool valid = rr < rows_per_cta && A < nn;
    double v[7] = {0, 0, 0, 0, 0, 0, 0};
    if (valid) {
        // two records per iteration (fixed order: q, then q+1) so 14 loads are in flight
        const int tile = n / T, t = n - tile * T;
        const double* base = partial + (long)tile * npairs * 7 * T + t;
        int q = npart_ptr[A];
        const int q1 = npart_ptr[A + 1];
        for (; q + 1 < q1; q += 2) {
            const double* p0 = base + (long)__ldg(npart + q) * 7 * T;
            const double* p1 = base + (long)__ldg(npart + q + 1) * 7 * T;
            double x0[7], x1[7];
#pragma unroll
            for (int cc = 0; cc < 7; ++cc) {
                x0[cc] = __ldcs(p0 + cc * T);
                x1[cc] = __ldcs(p1 + cc * T);
            }
#pragma unroll
            for (int cc = 0; cc < 7; ++cc)
                v[cc] = (v[cc] + x0[cc]) + x1[cc];
        }
        if (q < q1) {
            const double* p0 = base + (long)__ldg(npart + q) * 7 * T;
#pragma unroll
            for (int cc = 0; cc < 7; ++cc)
                v[cc] += __ldcs(p0 + cc * T);
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
            ss[(rr * 3 + i) * N + n] = v[4 + i];
    }
    __syncthreads();
    if (!valid)
        return;
    double* out = r + A * 4 * N + n;
    if (dir[A]) {
        out[0] = 0.0;
        out[N] = 0.0;
        out[2 * N] = 0.0;
    } else {
        const double* h = sH + n * N;
        const double* s0 = ss + rr * 3 * N;
        double h0 = 0.0, h1 = 0.0, h2 = 0.0;
        for (int m = 0; m < N; ++m) {
            h0 += h[m] * s0[m];
            h1 += h[m] * s0[N + m];
            h2 += h[m] * s0[2 * N + m];
        }
        out[0] = v[0] - h0;
        out[N] = v[1] - h1;
        out[2 * N] = v[2] - h2;
    }
    out[3 * N] = v[3];
}

void launch_residual_nodes(const double* H, int N, int nn, const int* npart_ptr, const int* npart,
                           const double* partial, const uint8_t* dir, double* r, int T,
                           long npairs, cudaStream_t st) {
    if (nn <= 0)
        return;
    const int rows = N >= 256 ? 1 : 256 / N;
    const size_t smem = sizeof(double) * ((size_t)N * N + 3 * (size_t)N * rows);
    note_launch();
    residual_nodes_kernel<<<(nn + rows - 1) / rows, rows * N, smem, st>>>(H, N, nn, rows, npart_ptr,
                                                                         npart, partial, dir, r, T, npairs);
}

// Neumann traction + backflow (assembly.cpp:376-413), node-centric: one
// thread per (boundary node, n) sums its incident facets in the reference's
// order (Neumann entry, then facet).  Dirichlet nodes are skipped because
// their velocity rows end at zero (assembly.cpp:541-544).
__global__ void boundary_kernel(BoundaryArgs a) {
    const int N = a.N;
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int bn = (int)(t / N);
    const int n = (int)(t - (long)bn * N);
    if (bn >= a.nbnodes)
        return;
    const int A = a.bnode[bn];
    if (a.dir[A])
        return;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int k = a.bptr[bn]; k < a.bptr[bn + 1]; ++k) {
        const int f = a.binc[k] >> 2, v = a.binc[k] & 3;
        const int f0 = a.fac[3 * f], f1 = a.fac[3 * f + 1], f2 = a.fac[3 * f + 2];
        const double nv[3] = {a.fnormal[3 * f], a.fnormal[3 * f + 1], a.fnormal[3 * f + 2]};
        const double w = a.farea[f] / 3.0;
        const double hn = a.h[(long)a.fbc[f] * N + n];
        double uf[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            uf[0][i] = a.state[((long)f0 * 4 + i) * N + n];
            uf[1][i] = a.state[((long)f1 * 4 + i) * N + n];
            uf[2][i] = a.state[((long)f2 * 4 + i) * N + n];
        }
        for (int q = 0; q < 3; ++q) {
            double uq[3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
                uq[i] = (q == 0 ? 2.0 / 3.0 : 1.0 / 6.0) * uf[0][i] +
                        (q == 1 ? 2.0 / 3.0 : 1.0 / 6.0) * uf[1][i] +
                        (q == 2 ? 2.0 / 3.0 : 1.0 / 6.0) * uf[2][i];
            const double un = uq[0] * nv[0] + uq[1] * nv[1] + uq[2] * nv[2];
            const double neg = un < 0.0 ? un : 0.0;
            const double sa = (q == v) ? 2.0 / 3.0 : 1.0 / 6.0;
#pragma unroll
            for (int i = 0; i < 3; ++i)
                acc[i] += w * sa * (-hn * nv[i] - 0.5 * a.rho * a.beta * neg * uq[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
        a.r[((long)A * 4 + i) * N + n] += acc[i];
}

void launch_boundary(const BoundaryArgs& a, cudaStream_t st) {
    if (a.nbnodes <= 0)
        return;
    const long threads = (long)a.nbnodes * a.N;
    note_launch();
    boundary_kernel<<<(int)((threads + 255) / 256), 256, 0, st>>>(a);
}

// Resistance outlets (BASELINE config 3; new physics, not in the reference —
// SURVEY 8(f) row 4; restated in oracle/hbgls_oracle.c): CTA (patch, sample n)
// forms the outward flux Q = sum_k b_k . v_k(n) over the patch's nodes in a
// fixed order (b_k = sum over the node's facets of area/3 * normal, the exact
// 3-point-rule weights) and adds R Q b_k to the velocity rows of its free
// nodes, optionally output-scaled (the GMRES operator S L S).  free_cols: only
// free nodes enter Q (the tangent's masked columns); the residual uses all.
__global__ void resistance_kernel(const int* __restrict__ ptr, const int* __restrict__ node,
                                  const double* __restrict__ b, const double* __restrict__ R,
                                  const uint8_t* __restrict__ dir, int N, const double* __restrict__ v,
                                  double* __restrict__ out, const double* __restrict__ scale, int free_cols,
                                  const int* skip) {
    if (skip && *skip)
        return;
    __shared__ double red[8];
    __shared__ double s_q;
    const int pch = blockIdx.x, n = blockIdx.y;
    const int k0 = ptr[pch], k1 = ptr[pch + 1];
    double acc = 0.0;
    for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const long A = node[k];
        if (free_cols && dir[A])
            continue;
        const double* vb = v + (A * 4) * N + n;
        acc += b[3 * k] * vb[0] + b[3 * k + 1] * vb[N] + b[3 * k + 2] * vb[2 * N];
    }
    for (int o = 16; o > 0; o >>= 1)
        acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double q = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            q += red[w];
        s_q = R[pch] * q;
    }
    __syncthreads();
    const double rq = s_q;
    for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const long A = node[k];
        if (dir[A])
            continue;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const long o = (A * 4 + i) * N + n;
            out[o] += (scale ? scale[o] : 1.0) * rq * b[3 * k + i];
        }
    }
}

void launch_resistance(const int* ptr, const int* node, const double* b, const double* R, int npatch,
                       const uint8_t* dir, int N, const double* v, double* out, const double* scale, int free_cols,
                       const int* skip, cudaStream_t st) {
    if (npatch <= 0)
        return;
    note_launch();
    resistance_kernel<<<dim3(npatch, N), 256, 0, st>>>(ptr, node, b, R, dir, N, v, out, scale, free_cols, skip);
}

// jacobi_preconditioner (linalg.cpp:130-154)
__global__ void jacobi_kernel(const double* __restrict__ vals, const int* __restrict__ diag_blk,
                              int nn, int N, double* __restrict__ inv, int* degenerate) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long total = (long)nn * 4 * N;
    if (t >= total)
        return;
    const long A = t / (4L * N);
    const int rem = (int)(t - A * 4 * N);
    const int c = rem / N, n = rem - c * N;
    const double d = vals[((long)diag_blk[A] * 8 + (c < 3 ? 0 : 7)) * N + n];
    if (fabs(d) < 1e-30) {
        inv[t] = 1.0;
        atomicAdd(degenerate, 1);
    } else {
        inv[t] = 1.0 / d;
    }
}

void launch_jacobi(const double* vals, const int* diag_blk, int nn, int N, double* inv_diag,
                   int* degenerate, cudaStream_t st) {
    const long total = (long)nn * 4 * N;
    if (total <= 0)
        return;
    note_launch();
    jacobi_kernel<<<(int)((total + 255) / 256), 256, 0, st>>>(vals, diag_blk, nn, N, inv_diag,
                                                              degenerate);
}

// ---------------------------------------------------------------- state ops

__global__ void install_dirichlet_kernel(const double* __restrict__ g, const uint8_t* dir, int nn,
                                         int N, double* state) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 3L * nn * N)
        return;
    const long A = t / (3L * N);
    if (!dir[A])
        return;
    const int rem = (int)(t - A * 3 * N);
    state[A * 4 * N + rem] = g[t];
}

void launch_install_dirichlet(const double* g, const uint8_t* dir, int nn, int N, double* state,
                              cudaStream_t st) {
    const long tot = 3L * nn * N;
    if (tot <= 0)
        return;
    note_launch();
    install_dirichlet_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(g, dir, nn, N, state);
}

__global__ void fill_pressure_kernel(double p0, int nn, int N, double* state) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long)nn * N)
        return;
    const long A = t / N;
    state[A * 4 * N + 3 * N + (t - A * N)] = p0;
}

void launch_fill_pressure(double p0, int nn, int N, double* state, cudaStream_t st) {
    const long tot = (long)nn * N;
    if (tot <= 0)
        return;
    note_launch();
    fill_pressure_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(p0, nn, N, state);
}

// y -= x except constrained velocity (hb_solver.cpp:205-215)
__global__ void newton_update_kernel(const double* __restrict__ dx, const uint8_t* dir, int nn,
                                     int N, double* state) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 4L * nn * N)
        return;
    const long A = t / (4L * N);
    const int c = (int)((t - A * 4 * N) / N);
    if (dir[A] && c < 3)
        return;
    state[t] -= dx[t];
}

void launch_newton_update(const double* dx, const uint8_t* dir, int nn, int N, double* state,
                          cudaStream_t st) {
    const long tot = 4L * nn * N;
    if (tot <= 0)
        return;
    note_launch();
    newton_update_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(dx, dir, nn, N, state);
}

// ---------------------------------------------------------------- vectors

__global__ void sqrt_abs_kernel(const double* in, double* out, long n) {
    for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (long)gridDim.x * blockDim.x)
        out[k] = sqrt(fabs(in[k]));
}
void launch_sqrt_abs(const double* in, double* out, long n, cudaStream_t st) {
    note_launch();
    sqrt_abs_kernel<<<4 * 148, 256, 0, st>>>(in, out, n);
}

__global__ void mul_kernel(const double* a, const double* b, double* out, long n) {
    for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (long)gridDim.x * blockDim.x)
        out[k] = a[k] * b[k];
}
void launch_mul(const double* a, const double* b, double* out, long n, cudaStream_t st) {
    note_launch();
    mul_kernel<<<4 * 148, 256, 0, st>>>(a, b, out, n);
}

__global__ void scaled_diff_kernel(const double* s, const double* a, const double* b, double* out,
                                   long n) {
    for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (long)gridDim.x * blockDim.x)
        out[k] = s[k] * (a[k] - b[k]);
}
void launch_scaled_diff(const double* s, const double* a, const double* b, double* out, long n,
                        cudaStream_t st) {
    note_launch();
    scaled_diff_kernel<<<4 * 148, 256, 0, st>>>(s, a, b, out, n);
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0)
        red[wid] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k)
            s += red[k];
    return s;  // valid in thread 0
}

// Fixed partition of [0,n) into kRedBlocks contiguous chunks.
__global__ void __launch_bounds__(kRedThreads) multidot_kernel(const double* __restrict__ V,
                                                               long ld, int nv,
                                                               const double* __restrict__ w,
                                                               long n, double* partial) {
    __shared__ double red[kRedThreads / 32];
    const long chunk = (n + kRedBlocks - 1) / kRedBlocks;
    const long lo = (long)blockIdx.x * chunk;
    const long hi = lo + chunk < n ? lo + chunk : n;
    for (int i = 0; i < nv; ++i) {
        const double* vi = V + (long)i * ld;
        double acc = 0.0;
        for (long k = lo + threadIdx.x; k < hi; k += blockDim.x)
            acc += vi[k] * w[k];
        const double s = block_sum(acc, red);
        if (threadIdx.x == 0)
            partial[(long)i * kRedBlocks + blockIdx.x] = s;
    }
}
void launch_multidot(const double* V, long ld, int nv, const double* w, long n, double* partial,
                     cudaStream_t st) {
    note_launch();
    multidot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(V, ld, nv, w, n, partial);
}

__global__ void reduce_partials_kernel(const double* __restrict__ partial, double* out,
                                       int take_sqrt, const int* skip, int nparts) {
    if (skip && *skip)
        return;
    __shared__ double red[kRedThreads / 32];
    const double* p = partial + (long)blockIdx.x * kRedBlocks;
    double acc = 0.0;
    for (int k = threadIdx.x; k < nparts; k += blockDim.x)
        acc += p[k];
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0)
        out[blockIdx.x] = (take_sqrt && blockIdx.x == 0) ? sqrt(s) : s;
}
void launch_reduce_partials(const double* partial, int nv, double* out, int take_sqrt,
                            cudaStream_t st, const int* skip, int nparts) {
    if (nv <= 0)
        return;
    note_launch();
    reduce_partials_kernel<<<nv, kRedThreads, 0, st>>>(partial, out, take_sqrt, skip, nparts);
}

// DFMA throughput probe: 16 independent FMA chains per thread, 32 warps per
// SM, a few ms of work (shorter runs under-read the peak by ~10% from the
// launch ramp).  Used by bench.py for the FP64 roofline peak (the driver's
// MEASURED_PEAKS.json has HBM and bf16 only).
constexpr int kPeakChains = 16;
__global__ void fp64_peak_kernel(double* out, int iters, double a, double b) {
    double x[kPeakChains];
#pragma unroll
    for (int k = 0; k < kPeakChains; ++k)
        x[k] = threadIdx.x * 1e-7 + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < kPeakChains; ++k)
            x[k] = fma(x[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kPeakChains; ++k)
        s += x[k];
    if (s == 12345.678)
        out[0] = s;
}

cudaError_t run_fp64_peak(int blocks, int threads, int iters, double* out, float* ms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fp64_peak_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);  // warm-up
    cudaEventRecord(e0);
    fp64_peak_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return err == cudaSuccess ? cudaGetLastError() : err;
}

}  // namespace hbgpu

namespace hbgpu {
cudaError_t residual_occupancy(int* blocks_per_sm, size_t smem, int T) {
    if (T == 4)
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, residual_chunk_kernel<4>, kChunkElems * 4, smem);
    if (T == 2)
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, residual_chunk_kernel<2>, kChunkElems * 2, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, residual_chunk_kernel<1>, kChunkElems, smem);
}
}  // namespace hbgpu
