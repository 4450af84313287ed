// Pointwise tangent P, persistent row pipeline (sm_100a, FP64).
//
// Replaces element_tangent_p + assemble_tangent (reference
// src/assembly.cpp:265-374, 550-666) for every block row.  Same arithmetic as
// the row kernel in hbgpu_tangent.cu (see the v5 comment there); what changes
// is how a row's operands reach shared memory:
//
//   * Each bucket row has a contiguous "row pack" in HBM, built at setup:
//       hdr   int4 {A, ninc, nblk, kdiag}, int4 {k0, nslots, dparts, afix}
//       sinfo int4 per phase-2 slot {c0, c1, j, bfix}
//       cols  int per block (column node), inc int2 per incidence
//       {e | la << 30, 4 x u8 block offsets}, cont u16 per contribution
//       (i << 2 | b, list order), blkc 8 doubles per block (n-invariant sums).
//     Dirichlet flags and blkc are (re)written on the device by
//     tangent_pack_refresh_kernel whenever the Dirichlet set changes.
//   * A persistent CTA walks rows r = blockIdx.x + k * gridDim.x.  Warp 0
//     streams them with bulk async copies (cp.async.bulk, the TMA engine's
//     1-D mode) completing on mbarriers: the pack of row k+1 lands during
//     phase 1 of row k, its gathers (each neighbour node's 4N state record,
//     each incidence's 20-double geometry record) during phase 2 of row k.
//     Two pack slots, one gather buffer.
//   * The compute of a row is three barrier-separated phases: contribution
//     records + per-(incidence, sample) summaries, per-(slot, sample)
//     accumulation, diagonal parts.  No global loads remain in them.
#include "hbgpu_internal.h"

#include <algorithm>

namespace hbgpu {

namespace {
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace

// ---------------------------------------------------------------- row packs

__host__ __device__ inline int pack_align16(int bytes) { return (bytes + 15) & ~15; }

// Byte offsets of the sections of a row pack.
struct PackSections {
    int sinfo, cols, inc, cont, blkc, total;
};
__host__ __device__ inline PackSections pack_sections(int ninc, int nblk, int nslots) {
    PackSections s;
    s.sinfo = 32;
    s.cols = s.sinfo + 16 * nslots;
    s.inc = s.cols + pack_align16(4 * nblk);
    s.cont = s.inc + pack_align16(8 * ninc);
    s.blkc = s.cont + pack_align16(2 * 4 * ninc);
    s.total = s.blkc + 64 * nblk;
    return s;
}

size_t tangent_pack_bytes(int ninc, int nblk) {
    const int dparts = (ninc + kTanPart - 1) / kTanPart;
    return (size_t)pack_sections(ninc, nblk, dparts + nblk - 1).total;
}

// Host: write the pack of one row (flags and blkc are left for the refresh
// kernel).  `cont` are the row's contributions in list order (i << 2 | b),
// `cptr` the row's per-block list offsets relative to the row start.
void tangent_pack_write(unsigned char* dst, int A, int k0, int ninc, int nblk, int kdiag,
                        const int* cols, const int2* inc, const uint16_t* cont, const int* cptr,
                        const uint8_t* order) {
    const int dparts = (ninc + kTanPart - 1) / kTanPart;
    const int nslots = dparts + nblk - 1;
    const PackSections s = pack_sections(ninc, nblk, nslots);
    std::fill(dst, dst + s.total, (unsigned char)0);
    int* h = reinterpret_cast<int*>(dst);
    h[0] = A;
    h[1] = ninc;
    h[2] = nblk;
    h[3] = kdiag;
    h[4] = k0;
    h[5] = nslots;
    h[6] = dparts;
    h[7] = 0;
    int* si = reinterpret_cast<int*>(dst + s.sinfo);
    for (int p = 0; p < dparts; ++p) {
        si[4 * p] = cptr[kdiag] + p * kTanPart;
        si[4 * p + 1] = std::min(cptr[kdiag] + (p + 1) * kTanPart, cptr[kdiag + 1]);
        si[4 * p + 2] = kdiag;
    }
    for (int q = 0; q + 1 < nblk; ++q) {
        const int j = order[q];
        si[4 * (dparts + q)] = cptr[j];
        si[4 * (dparts + q) + 1] = cptr[j + 1];
        si[4 * (dparts + q) + 2] = j;
    }
    std::copy(cols, cols + nblk, reinterpret_cast<int*>(dst + s.cols));
    std::copy(inc, inc + ninc, reinterpret_cast<int2*>(dst + s.inc));
    std::copy(cont, cont + 4 * ninc, reinterpret_cast<uint16_t*>(dst + s.cont));
}

// Device: Dirichlet flags (afix, bfix per slot) and block constants into the
// packs of one bucket; thread per row.
__global__ void tangent_pack_refresh_kernel(unsigned char* __restrict__ pack,
                                            const int* __restrict__ pack_ptr, int nrows,
                                            const uint8_t* __restrict__ dir,
                                            const double* __restrict__ blkc) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows)
        return;
    unsigned char* p = pack + (size_t)pack_ptr[r] * 16;
    int* h = reinterpret_cast<int*>(p);
    const int A = h[0], ninc = h[1], nblk = h[2], k0 = h[4], nslots = h[5];
    const PackSections s = pack_sections(ninc, nblk, nslots);
    h[7] = dir[A] != 0;
    int* si = reinterpret_cast<int*>(p + s.sinfo);
    const int* cols = reinterpret_cast<const int*>(p + s.cols);
    for (int q = 0; q < nslots; ++q)
        si[4 * q + 3] = dir[cols[si[4 * q + 2]]] != 0;
    double* bc = reinterpret_cast<double*>(p + s.blkc);
    for (int k = 0; k < 8 * nblk; ++k)
        bc[k] = blkc[(size_t)k0 * 8 + k];
}

void launch_tangent_pack_refresh(unsigned char* pack, const int* pack_ptr, int nrows,
                                 const uint8_t* dir, const double* blkc, cudaStream_t st) {
    if (nrows <= 0)
        return;
    note_launch();
    tangent_pack_refresh_kernel<<<(nrows + 127) / 128, 128, 0, st>>>(pack, pack_ptr, nrows, dir, blkc);
}

// ---------------------------------------------------------------- kernel

// contribution-record stride (doubles): 8 used, padded to 10 so the two records a
// warp's halves read in phase 2 do not fall on the same banks (TAN_REC_STRIDE)
// neighbour state records in shared memory: 4N doubles, padded (even, keeps the
// 16-byte bulk-copy alignment) to spread their bank offsets
#ifndef TAN_SU_PAD
#define TAN_SU_PAD 0
#endif
#ifndef TAN_SUMM_PAD
#define TAN_SUMM_PAD 0
#endif
#ifndef TAN_REC_STRIDE
#define TAN_REC_STRIDE 10
#endif
constexpr int kRecStride = TAN_REC_STRIDE;
// gathers of the next row issued by every warp (a few bulk copies each)
// instead of warp 0 alone, whose phase 2 then started late and held the
// row's closing barrier (ncu r2p: warp 0 spent 36% of its time issuing copies)
#ifndef TAN_GATHER_ALL
#define TAN_GATHER_ALL 1
#endif
// the row node's velocity comes from the four gathered element nodes (local
// slot 0 = the row node) instead of three more shared-memory loads
// phase-1 items of the single-sample kernels mapped with 16-lane-aligned sample groups per
// incidence (lanes past the last sample idle), so a half-warp never straddles incidences
#ifndef TAN_P1_ALIGN
#define TAN_P1_ALIGN 1
#endif
#ifndef TAN_UA_REUSE
#define TAN_UA_REUSE 1
#endif

// Sample pairs (P = 2): every phase-1 and phase-2 thread item covers a PAIR
// of consecutive time samples.  The geometry record, the contribution record
// and the index arithmetic are then loaded / computed once per two samples,
// the two samples' tau chains are independent (ILP), and the summaries and
// diagonal parts move as 16-byte double2 (sample stride padded to even).
// Used for the compile-time N of 5..19: at config 1 (N = 19) 0.858 -> 0.821 ms.
// At N = 47 the 512-thread CTA's items per row (ninc x 24 pairs vs ninc x 47)
// quantise worse and pairs lose (31.6 -> 32.8 ms, config 4), so N >= 31 and the
// generic kernel stay on single samples.
#ifndef TAN_PAIR_MAXN
#define TAN_PAIR_MAXN 19
#endif
#ifndef TAN_GRP_MINN
#define TAN_GRP_MINN 31
#endif
__host__ __device__ constexpr int tan_pair(int NC) { return (NC >= 3 && NC <= TAN_PAIR_MAXN) ? 2 : 1; }
// Phase-2 sample groups (single-sample kernels, NC >= 31): a phase-2 item is a
// block slot and G2 samples t, t + Q, t + 2Q, ... (Q = ceil(N / G2)), so the
// contribution record (4 x LDS.128, >= 2 wavefronts each even when broadcast) is
// read once per G2 samples; consecutive lanes still take consecutive samples,
// so summary loads and P stores stay contiguous per warp.  Phase 2 is bound by
// shared-memory bandwidth (ncu r2p: 100% of the wavefront rate, FP64 pipe 31%).
// G2 = ceil(N / 16): 16 lanes per slot, so a warp is exactly two slots (record loads are
// two broadcasts, summary loads two 128-byte runs).  Config-4 tangent at N = 31: G2 = 1 /
// 2 / 3 / 4 -> 21.0 / 18.2 / 22.0 / 22.2 ms (profiles/r3i_kbench_n31.log); at N = 47:
// 31.6 (G2 = 1) / 29.3 / 27.5 / 33.6 ms (r2q).  TAN_G2 > 0 forces a value (A/B builds).
#ifndef TAN_G2
#define TAN_G2 0
#endif
__host__ __device__ constexpr int tan_grp(int NC) {
    return (NC >= TAN_GRP_MINN) ? (TAN_G2 > 0 ? TAN_G2 : (NC + 15) / 16) : 1;
}
__host__ __device__ inline int tan_ntp(int NT, int P) { return (NT + P - 1) / P * P; }

struct PipeSmem {
    int meta, su, tg, summ, rec, dpart, mbar, total;  // byte offsets
};
__host__ __device__ inline PipeSmem pipe_layout(int max_pack, int mi, int max_blk, int N, int NT, int P) {
    PipeSmem L;
    const int dpmax = (mi + kTanPart - 1) / kTanPart;
    const int NTp = tan_ntp(NT, P);
    L.meta = 0;                                                   // 2 x max_pack
    L.su = L.meta + 2 * pack_align16(max_pack);                   // [blk][4N]
    L.tg = L.su + max_blk * (4 * N + TAN_SU_PAD) * 8;             // [inc][20]
    L.summ = L.tg + mi * kTGeo * 8;                               // [c][i][NTp]
    L.rec = L.summ + ((mi * 7 * (NTp + TAN_SUMM_PAD) + 1) & ~1) * 8;  // [p][10]
    L.dpart = L.rec + 4 * mi * kRecStride * 8;                    // [part][8][NTp]
    L.mbar = pack_align16(L.dpart + dpmax * 8 * NTp * 8);         // 3 mbarriers
    L.total = L.mbar + 32;
    return L;
}

static bool pipe_nc_listed(int N);
size_t tangent_pipe_smem(int max_pack, int max_inc, int max_blk, int N, int NT) {
    // the compile-time-N kernel (whole series per CTA) may use sample pairs
    const int P = (NT == N && pipe_nc_listed(N)) ? tan_pair(N) : 1;
    return (size_t)pipe_layout(max_pack, max_inc, max_blk, N, NT, P).total;
}

// THREADS per CTA (32 ... 512) is chosen per valence bucket from the row's
// work (incidences x samples) and the shared memory its summaries need.
// NC > 0: the time-sample count is the compile-time constant NC (and the
// whole series is one tile), so every N-strided shared/global address folds
// to an immediate offset; NC = 0 is the generic kernel.
template <int TAU, int THREADS, int NC>
__global__ void __launch_bounds__(THREADS, 512 / THREADS) tangent_pipe_kernel(TangentArgs a, PipeArgs pa) {
    constexpr int P = tan_pair(NC);
    constexpr bool UA = TAN_UA_REUSE && P == 1;  // (pairs: the six live doubles spill)
    extern __shared__ __align__(128) unsigned char smraw[];
    const int N = NC ? NC : a.N, NT = NC ? NC : a.NT;
    const int n0 = NC ? 0 : blockIdx.y * NT, nt = NC ? NC : min(NT, N - n0);
    const int NTp = tan_ntp(NT, P);
    const int nq = (nt + P - 1) / P;  // sample groups of this tile
    const PipeSmem Ls = pipe_layout(pa.max_pack, a.max_inc, a.max_blk, N, NT, P);
    // summaries, component-major [c][i][t]: the stores of one phase-1 pass are contiguous
    const int SI = NTp + TAN_SUMM_PAD, SC = a.max_inc * SI;
    const int mpack = pack_align16(pa.max_pack);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smraw + Ls.mbar);  // [0..1] packs, [2] gathers
    double* summ = reinterpret_cast<double*>(smraw + Ls.summ);
    double* rec = reinterpret_cast<double*>(smraw + Ls.rec);
    double* dpart = reinterpret_cast<double*>(smraw + Ls.dpart);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double rho = a.rho, diffc = 3.0 * a.nu * a.nu, dAB = kQA - kQB;
    const double c1 = kQB * (1.0 + dAB), c2 = dAB * dAB;
    const double mu = a.mu, pc = a.pseudo_c;
    const double inv_rho = 1.0 / rho;  // once per thread (w / rho per item was a full FP64 division)
    const int r0 = blockIdx.x, rs = gridDim.x, nrows = pa.nrows;
    if (threadIdx.x == 0) {
        for (int k = 0; k < 3; ++k)
            mbar_init(mbar + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue_pack = [&](int r, int slot) {  // warp 0, lane 0
        const int p0 = __ldg(pa.pack_ptr + r), p1 = __ldg(pa.pack_ptr + r + 1);
        const uint32_t bytes = (uint32_t)(p1 - p0) * 16u;
        mbar_expect_tx(mbar + slot, bytes);
        bulk_g2s(smraw + Ls.meta + slot * mpack, pa.pack + (size_t)p0 * 16, bytes, mbar + slot);
    };
    // copies idx = first, first + stride, ... of the row in pack slot `slot`:
    // idx < nblk the neighbour node's 4N state record, else an incidence's
    // geometry record.  `expect` (one thread per row) arms the mbarrier with the
    // row's byte count; its tx-count may run negative until then.
    auto issue_gather = [&](int slot, int first, int stride, bool expect) {
        const unsigned char* m = smraw + Ls.meta + slot * mpack;
        const int* h = reinterpret_cast<const int*>(m);
        const int ninc = h[1], nblk = h[2];
        const PackSections s = pack_sections(ninc, nblk, h[5]);
        const int* cols = reinterpret_cast<const int*>(m + s.cols);
        const int2* inc = reinterpret_cast<const int2*>(m + s.inc);
        double* su = reinterpret_cast<double*>(smraw + Ls.su);
        double* tg = reinterpret_cast<double*>(smraw + Ls.tg);
        if (expect)
            mbar_expect_tx(mbar + 2, (uint32_t)(nblk * 4 * N * 8 + ninc * kTGeo * 8));
        __syncwarp();
        for (int idx = first; idx < nblk + ninc; idx += stride) {
            if (idx < nblk) {
                bulk_g2s(su + (size_t)idx * (4 * N + TAN_SU_PAD), a.state + (size_t)cols[idx] * 4 * N, 4 * N * 8,
                         mbar + 2);
            } else {
                const int i = idx - nblk;
                bulk_g2s(tg + (size_t)i * kTGeo, a.tgeom + (size_t)(inc[i].x & 0x3FFFFFFF) * kTGeo, kTGeo * 8,
                         mbar + 2);
            }
        }
    };

    // prologue: pack and gathers of row 0
    if (warp == 0 && r0 < nrows) {
        if (lane == 0)
            issue_pack(r0, 0);
        mbar_wait(mbar + 0, 0);
        issue_gather(0, lane, 32, lane == 0);
    }

    // work items (x, q): x = incidence (phase 1) or slot (phase 2), q = sample group
    const int dx = blockDim.x / nq, dq = blockDim.x - dx * nq;
    const int x_start = threadIdx.x / nq, q_start = threadIdx.x - x_start * nq;
    // Diagonal block of the previous row: sum its parts in order, identity K on
    // Dirichlet rows (assembly.cpp:659-665).  Deferred into the next row's first
    // region so a row costs two barriers, not three.
    long pd_blk = -1;
    int pd_parts = 0;
    bool pd_fix = false;
    auto diag_sum = [&]() {
        if (pd_blk < 0)
            return;
        for (int it = threadIdx.x; it < 8 * nt; it += blockDim.x) {
            const int sl = it / nt, t = it - sl * nt, n = n0 + t;
            double v = 0.0;
            for (int p = 0; p < pd_parts; ++p)
                v += dpart[((size_t)p * 8 + sl) * NTp + t];
            if (sl == 0 && pd_fix)
                v = 1.0;
            __stcs(a.pvals + (pd_blk * 8 + sl) * N + n, v);
        }
    };
    int k = 0;
    for (int r = r0; r < nrows; r += rs, ++k) {
        // Pipeline: the pack of row k+1 is fetched during phase 1 of row k, its
        // gathers (into the single gather buffer, dead once phase 1 has read
        // it) during phase 2 and the diagonal pass of row k.
        const int ms = k & 1;
        const bool more = r + rs < nrows;
        if (warp == 0 && lane == 0 && more)
            issue_pack(r + rs, ms ^ 1);
        mbar_wait(mbar + ms, (k >> 1) & 1);  // pack landed (acquire for every thread)
        mbar_wait(mbar + 2, k & 1);           // gathers landed

        const unsigned char* m = smraw + Ls.meta + ms * mpack;
        const int* h = reinterpret_cast<const int*>(m);
        const int ninc = h[1], nblk = h[2], kdiag = h[3], k0 = h[4], nslots = h[5], dparts = h[6];
        const bool afix = h[7] != 0;
        const PackSections s = pack_sections(ninc, nblk, nslots);
        const int4* sinfo = reinterpret_cast<const int4*>(m + s.sinfo);
        const int2* inc = reinterpret_cast<const int2*>(m + s.inc);
        const uint16_t* cont = reinterpret_cast<const uint16_t*>(m + s.cont);
        const double* blkc = reinterpret_cast<const double*>(m + s.blkc);
        const double* su = reinterpret_cast<const double*>(smraw + Ls.su);
        const double* tg = reinterpret_cast<const double*>(smraw + Ls.tg);

        // ---- diagonal block of the previous row (its parts are in dpart)
        diag_sum();
        // ---- contribution records {dN_a (3), gg, dN_b (3), summary offset}
        for (int p = threadIdx.x; p < 4 * ninc; p += blockDim.x) {
            const int ent = cont[p];
            const int i = ent >> 2, b = ent & 3;
            const int la = (unsigned)inc[i].x >> 30;
            const double* gi = tg + i * kTGeo;
            const double ga0 = gi[3 * la], ga1 = gi[3 * la + 1], ga2 = gi[3 * la + 2];
            const double gb0 = gi[3 * b], gb1 = gi[3 * b + 1], gb2 = gi[3 * b + 2];
            double2* o = reinterpret_cast<double2*>(rec + p * kRecStride);
            o[0] = make_double2(ga0, ga1);
            o[1] = make_double2(ga2, fma(ga0, gb0, fma(ga1, gb1, ga2 * gb2)));
            o[2] = make_double2(gb0, gb1);
            o[3] = make_double2(gb2, __longlong_as_double((long long)i * SI));
        }
        // ---- phase 1: per (incidence, sample group) summaries
        bool bad_acc = false;
        auto p1item = [&](int i, int t) {
            const double* gi = tg + i * kTGeo;
            const int2 ic = inc[i];
            const int la = (unsigned)ic.x >> 30;
            const unsigned cols = (unsigned)ic.y;
            const double2 xv = *reinterpret_cast<const double2*>(gi + 12);  // V, xi00
            const double2 x1 = *reinterpret_cast<const double2*>(gi + 14);  // xi01, xi02
            const double2 x2 = *reinterpret_cast<const double2*>(gi + 16);  // xi11, xi12
            const double2 x3 = *reinterpret_cast<const double2*>(gi + 18);  // xi22, xi:xi
            const double x01 = 2.0 * x1.x, x02 = 2.0 * x1.y, x12 = 2.0 * x2.y, diff = diffc * x3.y;
            const double ga[3] = {gi[3 * la], gi[3 * la + 1], gi[3 * la + 2]};
            const double V = xv.x, w = 0.25 * V;
            auto quad = [&](const double v[3]) {
                const double q0 = fma(x02, v[2], fma(x01, v[1], xv.y * v[0]));
                const double q1 = fma(x12, v[2], x2.x * v[1]);
                return fma(v[0], q0, fma(v[1], q1, fma(v[2], x3.x * v[2], diff)));
            };
            int tt[P];
#pragma unroll
            for (int k2 = 0; k2 < P; ++k2)
                tt[k2] = min(t + k2, nt - 1);  // the padded sample repeats the last one (not stored past N)
            double u[P][4][3], usum[P][3];
#pragma unroll
            for (int k2 = 0; k2 < P; ++k2) {
                usum[k2][0] = usum[k2][1] = usum[k2][2] = 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    // UA: slot 0 = the row node (the quadrature sums are symmetric)
                    const int bb = UA ? ((la + b) & 3) : b;
                    const double* sb =
                        su + (size_t)((cols >> (8 * bb)) & 0xFFu) * (4 * N + TAN_SU_PAD) + n0 + tt[k2];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        u[k2][b][c] = sb[c * N];
                        usum[k2][c] += u[k2][b][c];
                    }
                }
            }
            bool bad = false;
            double tau_mean[P];
#pragma unroll
            for (int k2 = 0; k2 < P; ++k2) {
                tau_mean[k2] = 0.0;
                if (TAU == 1) {
                    const double um[3] = {0.25 * usum[k2][0], 0.25 * usum[k2][1], 0.25 * usum[k2][2]};
                    const double arg = quad(um);
                    const bool bm = !(arg > 0.0);
                    bad |= bm;
                    tau_mean[k2] = tau_or_zero(arg, bm);
                }
            }
            double tsum[P], z[P][3], kap[P][3];
#pragma unroll
            for (int k2 = 0; k2 < P; ++k2) {
                tsum[k2] = 0.0;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    z[k2][c] = kap[k2][c] = 0.0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
#pragma unroll
                for (int k2 = 0; k2 < P; ++k2) {
                    double uq[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        uq[c] = fma(dAB, u[k2][q][c], kQB * usum[k2][c]);
                    double tq = tau_mean[k2];
                    if (TAU == 0) {
                        const double arg = quad(uq);
                        const bool bq = !(arg > 0.0);
                        bad |= bq;
                        tq = tau_or_zero(arg, bq);
                    }
                    const double tadv = tq * fma(uq[0], ga[0], fma(uq[1], ga[1], uq[2] * ga[2]));
                    tsum[k2] += tq;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        z[k2][c] = fma(tq, uq[c], z[k2][c]);
                        kap[k2][c] = fma(tadv, uq[c], kap[k2][c]);
                    }
                }
            }
            // + sum_q N_a(q) u_q = B usum + (A-B) u_{q=a} = c1 usum + c2 u_A (u_A: the row node)
            const double wr = w * rho, wo = w * inv_rho;
            double o[7][P];
#pragma unroll
            for (int k2 = 0; k2 < P; ++k2) {
                const double* sA = su + (size_t)kdiag * (4 * N + TAN_SU_PAD) + n0 + tt[k2];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double uA = UA ? u[k2][0][c] : sA[c * N];
                    o[c][k2] = wr * fma(c1, usum[k2][c], fma(c2, uA, kap[k2][c]));
                    o[3 + c][k2] = w * z[k2][c];
                }
                o[6][k2] = wo * tsum[k2];
            }
            bad_acc |= bad;
            double* so = summ + (size_t)i * SI + t;
#pragma unroll
            for (int c = 0; c < 7; ++c) {
                if (P == 2)
                    *reinterpret_cast<double2*>(so + c * SC) = make_double2(o[c][0], o[c][P - 1]);
                else
                    so[c * SC] = o[c][0];
            }
        };
        if constexpr (TAN_P1_ALIGN && P == 1 && NC >= TAN_GRP_MINN) {  // (N = 1: 16x the loop trips)
            const int nqa = (nq + 15) & ~15;
            for (int it = threadIdx.x; it < ninc * nqa; it += blockDim.x) {
                const int i = it / nqa, q = it - i * nqa;
                if (q < nq)
                    p1item(i, q);
            }
        } else {
            for (int it = threadIdx.x, i = x_start, q = q_start; it < ninc * nq;
                 it += blockDim.x, q += dq, i += dx + (q >= nq), q -= (q >= nq ? nq : 0))
                p1item(i, P * q);
        }
        if (bad_acc)
            atomicOr(a.flag, 1);
        __syncthreads();

#if TAN_GATHER_ALL
        if (more) {  // every warp issues a few of the next row's copies
            mbar_wait(mbar + (ms ^ 1), ((k + 1) >> 1) & 1);
            const int nw = blockDim.x >> 5;
            issue_gather(ms ^ 1, lane * nw + warp, 32 * nw, threadIdx.x == 0);
        }
#else
        if (warp == 0 && more) {
            mbar_wait(mbar + (ms ^ 1), ((k + 1) >> 1) & 1);
            issue_gather(ms ^ 1, lane, 32, lane == 0);
        }
#endif
        // ---- phase 2: per (slot, sample group) register accumulation
        if constexpr (P == 1) {
            // item = (slot, q): samples q, q + Q2, ... (G2 of them); the contribution
            // record is read once per item
            constexpr int G2 = tan_grp(NC);
            const int Q2 = (nt + G2 - 1) / G2;
            const int dx2 = blockDim.x / Q2, dq2 = blockDim.x - dx2 * Q2;
            int slot = threadIdx.x / Q2, q = threadIdx.x - slot * Q2;
            for (int it = threadIdx.x; it < nslots * Q2;
                 it += blockDim.x, q += dq2, slot += dx2 + (q >= Q2), q -= (q >= Q2 ? Q2 : 0)) {
                const int4 info = sinfo[slot];
                const int j = info.z;
                const bool bfix = info.w != 0;
                int tk[G2];
#pragma unroll
                for (int g = 0; g < G2; ++g)
                    tk[g] = min(q + g * Q2, nt - 1);  // a padded sample repeats the last one (not stored)
                double K[G2], G0[G2], G1[G2], G2v[G2], D0[G2], D1[G2], D2[G2], L[G2];
#pragma unroll
                for (int g = 0; g < G2; ++g)
                    K[g] = G0[g] = G1[g] = G2v[g] = D0[g] = D1[g] = D2[g] = L[g] = 0.0;
                for (int p = info.x; p < info.y; ++p) {
                    const double2* rp = reinterpret_cast<const double2*>(rec + p * kRecStride);
                    const double2 ra = rp[0], rb = rp[1], rc = rp[2], rd = rp[3];
                    const double* sp = summ + __double_as_longlong(rd.y);
                    const double gb0 = rc.x, gb1 = rc.y, gb2 = rd.x;
#pragma unroll
                    for (int g = 0; g < G2; ++g) {
                        const double* sg = sp + tk[g];
                        const double s0 = sg[0], s1 = sg[SC], s2 = sg[2 * SC], s3 = sg[3 * SC], s4 = sg[4 * SC],
                                     s5 = sg[5 * SC], s6 = sg[6 * SC];
                        K[g] = fma(s0, gb0, fma(s1, gb1, fma(s2, gb2, K[g])));
                        const double al = fma(s3, ra.x, fma(s4, ra.y, s5 * rb.x));  // w alpha_a = (w z) . dN_a
                        G0[g] = fma(al, gb0, G0[g]);
                        G1[g] = fma(al, gb1, G1[g]);
                        G2v[g] = fma(al, gb2, G2v[g]);
                        const double alb = fma(s3, gb0, fma(s4, gb1, s5 * gb2));
                        D0[g] = fma(ra.x, alb, D0[g]);
                        D1[g] = fma(ra.y, alb, D1[g]);
                        D2[g] = fma(rb.x, alb, D2[g]);
                        L[g] = fma(rb.y, s6, L[g]);
                    }
                }
                if (slot >= dparts || slot == 0) {
                    const double2* bc = reinterpret_cast<const double2*>(blkc + j * 8);
                    const double2 b0 = bc[0], b1 = bc[1], b2 = bc[2], b3 = bc[3];
                    const double kc = fma(mu, b0.x, pc * b0.y);
#pragma unroll
                    for (int g = 0; g < G2; ++g) {
                        K[g] += kc;
                        G0[g] += b1.x;
                        G1[g] += b1.y;
                        G2v[g] += b2.x;
                        D0[g] += b2.y;
                        D1[g] += b3.x;
                        D2[g] += b3.y;
                    }
                }
#pragma unroll
                for (int g = 0; g < G2; ++g) {
                    if (afix || bfix)
                        K[g] = 0.0;
                    if (afix)
                        G0[g] = G1[g] = G2v[g] = 0.0;
                    if (bfix)
                        D0[g] = D1[g] = D2[g] = 0.0;
                }
#pragma unroll
                for (int g = 0; g < G2; ++g) {
                    const int t = q + g * Q2;
                    if (t >= nt)
                        break;
                    if (slot >= dparts) {
                        double* out = a.pvals + ((long)(k0 + j) * 8) * N + n0 + t;
                        __stcs(out, K[g]);
                        __stcs(out + N, G0[g]);
                        __stcs(out + 2 * N, G1[g]);
                        __stcs(out + 3 * N, G2v[g]);
                        __stcs(out + 4 * N, D0[g]);
                        __stcs(out + 5 * N, D1[g]);
                        __stcs(out + 6 * N, D2[g]);
                        __stcs(out + 7 * N, L[g]);
                    } else {
                        double* o = dpart + (size_t)slot * 8 * NTp + t;
                        o[0] = K[g];
                        o[NTp] = G0[g];
                        o[2 * NTp] = G1[g];
                        o[3 * NTp] = G2v[g];
                        o[4 * NTp] = D0[g];
                        o[5 * NTp] = D1[g];
                        o[6 * NTp] = D2[g];
                        o[7 * NTp] = L[g];
                    }
                }
            }
        } else {
            for (int it = threadIdx.x, slot = x_start, q = q_start; it < nslots * nq;
                 it += blockDim.x, q += dq, slot += dx + (q >= nq), q -= (q >= nq ? nq : 0)) {
                const int t = P * q;
                const int4 info = sinfo[slot];
                const int j = info.z;
                const bool bfix = info.w != 0;
                double K[P], G0[P], G1[P], G2[P], D0[P], D1[P], D2[P], L[P];
    #pragma unroll
                for (int k2 = 0; k2 < P; ++k2)
                    K[k2] = G0[k2] = G1[k2] = G2[k2] = D0[k2] = D1[k2] = D2[k2] = L[k2] = 0.0;
                for (int p = info.x; p < info.y; ++p) {
                    const double2* rp = reinterpret_cast<const double2*>(rec + p * kRecStride);
                    const double2 ra = rp[0], rb = rp[1], rc = rp[2], rd = rp[3];
                    const double* sp = summ + __double_as_longlong(rd.y) + t;
                    const double gb0 = rc.x, gb1 = rc.y, gb2 = rd.x;
                    double sv[7][P];
    #pragma unroll
                    for (int c = 0; c < 7; ++c) {
                        if (P == 2) {
                            const double2 v2 = *reinterpret_cast<const double2*>(sp + c * SC);
                            sv[c][0] = v2.x;
                            sv[c][P - 1] = v2.y;
                        } else {
                            sv[c][0] = sp[c * SC];
                        }
                    }
    #pragma unroll
                    for (int k2 = 0; k2 < P; ++k2) {
                        K[k2] = fma(sv[0][k2], gb0, fma(sv[1][k2], gb1, fma(sv[2][k2], gb2, K[k2])));
                        // w alpha_a = (w z) . dN_a
                        const double al = fma(sv[3][k2], ra.x, fma(sv[4][k2], ra.y, sv[5][k2] * rb.x));
                        G0[k2] = fma(al, gb0, G0[k2]);
                        G1[k2] = fma(al, gb1, G1[k2]);
                        G2[k2] = fma(al, gb2, G2[k2]);
                        const double alb = fma(sv[3][k2], gb0, fma(sv[4][k2], gb1, sv[5][k2] * gb2));
                        D0[k2] = fma(ra.x, alb, D0[k2]);
                        D1[k2] = fma(ra.y, alb, D1[k2]);
                        D2[k2] = fma(rb.x, alb, D2[k2]);
                        L[k2] = fma(rb.y, sv[6][k2], L[k2]);
                    }
                }
                if (slot >= dparts || slot == 0) {
                    const double2* bc = reinterpret_cast<const double2*>(blkc + j * 8);
                    const double2 b0 = bc[0], b1 = bc[1], b2 = bc[2], b3 = bc[3];
                    const double kc = fma(mu, b0.x, pc * b0.y);
    #pragma unroll
                    for (int k2 = 0; k2 < P; ++k2) {
                        K[k2] += kc;
                        G0[k2] += b1.x;
                        G1[k2] += b1.y;
                        G2[k2] += b2.x;
                        D0[k2] += b2.y;
                        D1[k2] += b3.x;
                        D2[k2] += b3.y;
                    }
                }
    #pragma unroll
                for (int k2 = 0; k2 < P; ++k2) {
                    if (afix || bfix)
                        K[k2] = 0.0;
                    if (afix)
                        G0[k2] = G1[k2] = G2[k2] = 0.0;
                    if (bfix)
                        D0[k2] = D1[k2] = D2[k2] = 0.0;
                }
                if (slot >= dparts) {
    #pragma unroll
                    for (int k2 = 0; k2 < P; ++k2) {
                        if (t + k2 >= nt)
                            break;
                        double* out = a.pvals + ((long)(k0 + j) * 8) * N + n0 + t + k2;
                        __stcs(out, K[k2]);
                        __stcs(out + N, G0[k2]);
                        __stcs(out + 2 * N, G1[k2]);
                        __stcs(out + 3 * N, G2[k2]);
                        __stcs(out + 4 * N, D0[k2]);
                        __stcs(out + 5 * N, D1[k2]);
                        __stcs(out + 6 * N, D2[k2]);
                        __stcs(out + 7 * N, L[k2]);
                    }
                } else {
                    double* o = dpart + (size_t)slot * 8 * NTp + t;
                    if (P == 2) {
                        *reinterpret_cast<double2*>(o) = make_double2(K[0], K[P - 1]);
                        *reinterpret_cast<double2*>(o + NTp) = make_double2(G0[0], G0[P - 1]);
                        *reinterpret_cast<double2*>(o + 2 * NTp) = make_double2(G1[0], G1[P - 1]);
                        *reinterpret_cast<double2*>(o + 3 * NTp) = make_double2(G2[0], G2[P - 1]);
                        *reinterpret_cast<double2*>(o + 4 * NTp) = make_double2(D0[0], D0[P - 1]);
                        *reinterpret_cast<double2*>(o + 5 * NTp) = make_double2(D1[0], D1[P - 1]);
                        *reinterpret_cast<double2*>(o + 6 * NTp) = make_double2(D2[0], D2[P - 1]);
                        *reinterpret_cast<double2*>(o + 7 * NTp) = make_double2(L[0], L[P - 1]);
                    } else {
                        o[0] = K[0];
                        o[NTp] = G0[0];
                        o[2 * NTp] = G1[0];
                        o[3 * NTp] = G2[0];
                        o[4 * NTp] = D0[0];
                        o[5 * NTp] = D1[0];
                        o[6 * NTp] = D2[0];
                        o[7 * NTp] = L[0];
                    }
                }
            }
        }
        __syncthreads();
        pd_blk = k0 + kdiag;
        pd_parts = dparts;
        pd_fix = afix;
    }
    diag_sum();
}

// Compile-time time-sample counts of the BASELINE configs (N = 2 Nm - 1).
#define HBGPU_PIPE_NC_LIST(X) X(1) X(5) X(7) X(19) X(31) X(47)
static bool pipe_nc_listed(int N) {
#define HBGPU_NC_IS(n) if (N == n) return true;
    HBGPU_PIPE_NC_LIST(HBGPU_NC_IS)
#undef HBGPU_NC_IS
    return false;
}

template <int T, int NC>
static cudaError_t configure_pipe_tn(int b) {
    cudaError_t e = cudaFuncSetAttribute(tangent_pipe_kernel<0, T, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e != cudaSuccess)
        return e;
    return cudaFuncSetAttribute(tangent_pipe_kernel<1, T, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

template <int T>
static cudaError_t configure_pipe_t(size_t bytes) {
    const int b = int(bytes < 48 * 1024 ? 48 * 1024 : bytes);
    cudaError_t e = configure_pipe_tn<T, 0>(b);
#define HBGPU_CFG_NC(n)            \
    if (e == cudaSuccess)          \
        e = configure_pipe_tn<T, n>(b);
    HBGPU_PIPE_NC_LIST(HBGPU_CFG_NC)
#undef HBGPU_CFG_NC
    return e;
}

cudaError_t configure_tangent_pipe_smem(int threads, size_t bytes) {
    switch (threads) {
    case 32: return configure_pipe_t<32>(bytes);
    case 64: return configure_pipe_t<64>(bytes);
    case 128: return configure_pipe_t<128>(bytes);
    case 256: return configure_pipe_t<256>(bytes);
    case 512: return configure_pipe_t<512>(bytes);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t tangent_pipe_occupancy(int threads, int* blocks_per_sm, size_t smem) {
    switch (threads) {
    case 32: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tangent_pipe_kernel<0, 32, 0>, 32, smem);
    case 64: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tangent_pipe_kernel<0, 64, 0>, 64, smem);
    case 128: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tangent_pipe_kernel<0, 128, 0>, 128, smem);
    case 256: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tangent_pipe_kernel<0, 256, 0>, 256, smem);
    case 512: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tangent_pipe_kernel<0, 512, 0>, 512, smem);
    default: return cudaErrorInvalidValue;
    }
}

template <int T, int NC>
static void launch_pipe_tn(const TangentArgs& a, const PipeArgs& p, dim3 grid, size_t smem, cudaStream_t st) {
    if (a.tau_mode == 1)
        tangent_pipe_kernel<1, T, NC><<<grid, T, smem, st>>>(a, p);
    else
        tangent_pipe_kernel<0, T, NC><<<grid, T, smem, st>>>(a, p);
}

template <int T>
static void launch_pipe_t(const TangentArgs& a, const PipeArgs& p, dim3 grid, size_t smem, cudaStream_t st) {
    if (a.NT == a.N) {
        switch (a.N) {
#define HBGPU_LAUNCH_NC(n) \
    case n:                \
        return launch_pipe_tn<T, n>(a, p, grid, smem, st);
            HBGPU_PIPE_NC_LIST(HBGPU_LAUNCH_NC)
#undef HBGPU_LAUNCH_NC
        default:
            break;
        }
    }
    launch_pipe_tn<T, 0>(a, p, grid, smem, st);
}

void launch_tangent_pipe(const TangentArgs& a, const PipeArgs& p, int threads, int grid_x, size_t smem,
                         cudaStream_t st) {
    if (p.nrows <= 0)
        return;
    note_launch();
    const dim3 grid(grid_x, (a.N + a.NT - 1) / a.NT);
    switch (threads) {
    case 32: launch_pipe_t<32>(a, p, grid, smem, st); break;
    case 64: launch_pipe_t<64>(a, p, grid, smem, st); break;
    case 256: launch_pipe_t<256>(a, p, grid, smem, st); break;
    case 512: launch_pipe_t<512>(a, p, grid, smem, st); break;
    default: launch_pipe_t<128>(a, p, grid, smem, st); break;
    }
}

}  // namespace hbgpu
