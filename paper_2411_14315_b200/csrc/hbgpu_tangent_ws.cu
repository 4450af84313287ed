// Pointwise tangent P, warp-split rows (sm_100a, FP64).
//
// Replaces element_tangent_p + assemble_tangent (reference
// src/assembly.cpp:265-374, 550-666) for the block rows of the
// compile-time-N buckets.  Same arithmetic and row packs as the persistent
// pipeline (hbgpu_tangent_pipe.cu); what changes is the work split inside a
// CTA.  The pipeline splits each phase of a row over ALL threads, so every row
// costs two CTA barriers, and at N = 47 (one 512-thread CTA per SM, 151 KB of
// shared memory per row) ncu attributes 31% of the warp-stall samples to those
// barriers: the (incidence, sample) and (slot, sample) items of a row quantise
// to 2-3 rounds of 512 threads.  Here every warp owns a fixed range of time
// samples of the CTA's current row and runs BOTH phases for them:
//   phase 1  lanes over (incidence, own sample): the 7 summaries into shared
//            memory (only this warp reads them back);
//   phase 2  lanes over (block slot, own sample): register accumulation, P
//            written once; the diagonal block's parts summed by the same warp.
// No CTA barrier remains.  Row data are shared through mbarriers and a
// counter: the row pack and the contribution records (3 slots), the
// neighbour state records and geometry (1 slot, released when every warp has
// finished phase 1 of the row: the last warp to finish issues the next row's
// gathers and the pack after that).  Contribution records {dN_a, dN_a.dN_b,
// dN_b, incidence} are mesh constants, built once at setup
// (tangent_recs_kernel) and bulk-copied per row.
#include "hbgpu_internal.h"

namespace hbgpu {

namespace {
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
__host__ __device__ inline int ws_align16(int bytes) { return (bytes + 15) & ~15; }
}  // namespace

// Row-pack sections (identical to hbgpu_tangent_pipe.cu's pack_sections).
struct WsPackSections {
    int sinfo, cols, inc, cont, blkc, total;
};
__host__ __device__ inline WsPackSections ws_pack_sections(int ninc, int nblk, int nslots) {
    WsPackSections s;
    s.sinfo = 32;
    s.cols = s.sinfo + 16 * nslots;
    s.inc = s.cols + ws_align16(4 * nblk);
    s.cont = s.inc + ws_align16(8 * ninc);
    s.blkc = s.cont + ws_align16(2 * 4 * ninc);
    s.total = s.blkc + 64 * nblk;
    return s;
}

// Contribution records of every row of a bucket, in the row's contribution
// list order: {dN_a (3), dN_a . dN_b, dN_b (3), incidence index}; rec_ptr[r] =
// first record of row r (4 x ninc per row).  Thread per row.
__global__ void tangent_recs_kernel(const unsigned char* __restrict__ pack, const int* __restrict__ pack_ptr,
                                    int nrows, const double* __restrict__ tgeom, const long* __restrict__ rec_ptr,
                                    double* __restrict__ recs) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows)
        return;
    const unsigned char* p = pack + (size_t)pack_ptr[r] * 16;
    const int* h = reinterpret_cast<const int*>(p);
    const int ninc = h[1], nblk = h[2], nslots = h[5];
    const WsPackSections s = ws_pack_sections(ninc, nblk, nslots);
    const int2* inc = reinterpret_cast<const int2*>(p + s.inc);
    const uint16_t* cont = reinterpret_cast<const uint16_t*>(p + s.cont);
    double* o = recs + rec_ptr[r] * 8;
    for (int q = 0; q < 4 * ninc; ++q) {
        const int i = cont[q] >> 2, b = cont[q] & 3;
        const unsigned ie = (unsigned)inc[i].x;
        const int la = ie >> 30;
        const double* g = tgeom + (size_t)(ie & 0x3FFFFFFF) * kTGeo;
        const double ga0 = g[3 * la], ga1 = g[3 * la + 1], ga2 = g[3 * la + 2];
        const double gb0 = g[3 * b], gb1 = g[3 * b + 1], gb2 = g[3 * b + 2];
        double* d = o + 8 * q;
        d[0] = ga0;
        d[1] = ga1;
        d[2] = ga2;
        d[3] = fma(ga0, gb0, fma(ga1, gb1, ga2 * gb2));
        d[4] = gb0;
        d[5] = gb1;
        d[6] = gb2;
        d[7] = __longlong_as_double((long long)i);
    }
}

void launch_tangent_recs(const unsigned char* pack, const int* pack_ptr, int nrows, const double* tgeom,
                         const long* rec_ptr, double* recs, cudaStream_t st) {
    if (nrows <= 0)
        return;
    note_launch();
    tangent_recs_kernel<<<(nrows + 127) / 128, 128, 0, st>>>(pack, pack_ptr, nrows, tgeom, rec_ptr, recs);
}

struct WsSmem {
    int meta, recs, su, tg, summ, dpart, ctl, total;  // byte offsets
};
// 3 pack / record slots, 1 gather slot (state records, geometry)
__host__ __device__ inline WsSmem ws_layout(int max_pack, int mi, int max_blk, int N) {
    WsSmem L;
    const int dpmax = (mi + kTanPart - 1) / kTanPart;
    L.meta = 0;
    L.recs = L.meta + 3 * ws_align16(max_pack);
    L.su = L.recs + 3 * 4 * mi * 64;                 // [blk][4N]
    L.tg = L.su + max_blk * 4 * N * 8;               // [inc][20]
    L.summ = L.tg + mi * kTGeo * 8;                  // [c][i][N]
    L.dpart = L.summ + ((mi * 7 * N + 1) & ~1) * 8;  // [part][8][N]
    L.ctl = ws_align16(L.dpart + dpmax * 8 * N * 8); // 3 pack mbarriers, 1 gather mbarrier, counter
    L.total = L.ctl + 64;
    return L;
}

size_t tangent_ws_smem(int max_pack, int max_inc, int max_blk, int N) {
    return (size_t)ws_layout(max_pack, max_inc, max_blk, N).total;
}

template <int TAU, int THREADS, int NC>
__global__ void __launch_bounds__(THREADS, 512 / THREADS) tangent_ws_kernel(TangentArgs a, PipeArgs pa,
                                                                            const double* __restrict__ recs_g,
                                                                            const long* __restrict__ rec_ptr) {
    constexpr int N = NC, W = THREADS / 32;
    extern __shared__ __align__(128) unsigned char smraw[];
    const WsSmem Ls = ws_layout(pa.max_pack, a.max_inc, a.max_blk, N);
    const int SI = N, SC = a.max_inc * SI;
    const int mpack = ws_align16(pa.max_pack), mrec = 4 * a.max_inc * 8;  // doubles per record slot
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smraw + Ls.ctl);  // [0..2] pack + records, [3] gathers
    int* counter = reinterpret_cast<int*>(smraw + Ls.ctl + 32);
    double* summ = reinterpret_cast<double*>(smraw + Ls.summ);
    double* dpart = reinterpret_cast<double*>(smraw + Ls.dpart);
    double* su = reinterpret_cast<double*>(smraw + Ls.su);
    double* tg = reinterpret_cast<double*>(smraw + Ls.tg);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double rho = a.rho, diffc = 3.0 * a.nu * a.nu, dAB = kQA - kQB;
    const double c1 = kQB * (1.0 + dAB), c2 = dAB * dAB;
    const double mu = a.mu, pc = a.pseudo_c;
    const int r0 = blockIdx.x, rs = gridDim.x, nrows = pa.nrows;
    // this warp's samples [t0, t1)
    const int t0 = (warp * N) / W, t1 = ((warp + 1) * N) / W, ns = t1 - t0;
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; ++k)
            mbar_init(mbar + k, 1);
        *counter = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue_pack = [&](int r, int slot) {  // one thread: row pack + contribution records
        const int p0 = __ldg(pa.pack_ptr + r), p1 = __ldg(pa.pack_ptr + r + 1);
        const uint32_t pbytes = (uint32_t)(p1 - p0) * 16u;
        const long q0 = __ldg(rec_ptr + r), q1 = __ldg(rec_ptr + r + 1);
        const uint32_t rbytes = (uint32_t)(q1 - q0) * 64u;
        mbar_expect_tx(mbar + slot, pbytes + rbytes);
        bulk_g2s(smraw + Ls.meta + slot * mpack, pa.pack + (size_t)p0 * 16, pbytes, mbar + slot);
        bulk_g2s(smraw + Ls.recs + slot * mrec * 8, recs_g + q0 * 8, rbytes, mbar + slot);
    };
    auto issue_gather = [&](int slot) {  // one warp: the row's neighbour state records and geometry
        const unsigned char* m = smraw + Ls.meta + slot * mpack;
        const int* h = reinterpret_cast<const int*>(m);
        const int ninc = h[1], nblk = h[2];
        const WsPackSections s = ws_pack_sections(ninc, nblk, h[5]);
        const int* cols = reinterpret_cast<const int*>(m + s.cols);
        const int2* inc = reinterpret_cast<const int2*>(m + s.inc);
        if (lane == 0)
            mbar_expect_tx(mbar + 3, (uint32_t)(nblk * 4 * N * 8 + ninc * kTGeo * 8));
        __syncwarp();
        for (int j = lane; j < nblk; j += 32)
            bulk_g2s(su + (size_t)j * 4 * N, a.state + (size_t)cols[j] * 4 * N, 4 * N * 8, mbar + 3);
        for (int i = lane; i < ninc; i += 32)
            bulk_g2s(tg + (size_t)i * kTGeo, a.tgeom + (size_t)(inc[i].x & 0x3FFFFFFF) * kTGeo, kTGeo * 8,
                     mbar + 3);
    };

    // prologue: packs of the first two rows, gathers of the first
    if (warp == 0 && r0 < nrows) {
        if (lane == 0) {
            issue_pack(r0, 0);
            if (r0 + rs < nrows)
                issue_pack(r0 + rs, 1);
        }
        mbar_wait(mbar + 0, 0);
        issue_gather(0);
    }

    int k = 0;
    bool bad_acc = false;
    for (int r = r0; r < nrows; r += rs, ++k) {
        const int ms = k % 3;
        mbar_wait(mbar + ms, (k / 3) & 1);  // pack + records of this row landed
        mbar_wait(mbar + 3, k & 1);          // its gathers landed

        const unsigned char* m = smraw + Ls.meta + ms * mpack;
        const int* h = reinterpret_cast<const int*>(m);
        const int ninc = h[1], nblk = h[2], kdiag = h[3], k0 = h[4], nslots = h[5], dparts = h[6];
        const bool afix = h[7] != 0;
        const WsPackSections s = ws_pack_sections(ninc, nblk, nslots);
        const int4* sinfo = reinterpret_cast<const int4*>(m + s.sinfo);
        const int2* inc = reinterpret_cast<const int2*>(m + s.inc);
        const double* blkc = reinterpret_cast<const double*>(m + s.blkc);
        const double* rec = reinterpret_cast<const double*>(smraw + Ls.recs) + ms * mrec;

        // ---- phase 1: (incidence, own sample) summaries
        for (int it = lane; it < ninc * ns; it += 32) {
            const int i = it / ns, t = t0 + (it - i * ns);
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
            double u[4][3], usum[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const double* sb = su + (size_t)((cols >> (8 * b)) & 0xFFu) * 4 * N + t;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    u[b][c] = sb[c * N];
                    usum[c] += u[b][c];
                }
            }
            bool bad = false;
            double tau_mean = 0.0;
            if (TAU == 1) {
                const double um[3] = {0.25 * usum[0], 0.25 * usum[1], 0.25 * usum[2]};
                const double arg = quad(um);
                bad = !(arg > 0.0);
                tau_mean = tau_or_zero(arg, bad);
            }
            double tsum = 0.0, z[3] = {0.0, 0.0, 0.0}, kap[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double uq[3];
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    uq[c] = fma(dAB, u[q][c], kQB * usum[c]);
                double tq = tau_mean;
                if (TAU == 0) {
                    const double arg = quad(uq);
                    const bool bq = !(arg > 0.0);
                    bad |= bq;
                    tq = tau_or_zero(arg, bq);
                }
                const double tadv = tq * fma(uq[0], ga[0], fma(uq[1], ga[1], uq[2] * ga[2]));
                tsum += tq;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    z[c] = fma(tq, uq[c], z[c]);
                    kap[c] = fma(tadv, uq[c], kap[c]);
                }
            }
            // + sum_q N_a(q) u_q = c1 usum + c2 u_A (u_A: the row node)
            const double* sA = su + (size_t)kdiag * 4 * N + t;
            bad_acc |= bad;
            double* so = summ + (size_t)i * SI + t;
            const double wr = w * rho;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                so[c * SC] = wr * fma(c1, usum[c], fma(c2, sA[c * N], kap[c]));
                so[(3 + c) * SC] = w * z[c];
            }
            so[6 * SC] = (w / rho) * tsum;
        }
        // phase 1 of this row done in this warp: the last warp to get here
        // releases the gather slot — next row's gathers, the pack after that
        {
            int last = 0;
            __threadfence_block();  // this warp's reads of the gather slot precede its arrival
            if (lane == 0)
                last = atomicAdd(counter, 1) == (k + 1) * W - 1;
            last = __shfl_sync(0xFFFFFFFFu, last, 0);
            if (last) {
                __threadfence_block();
                if (r + rs < nrows) {
                    const int ns1 = (k + 1) % 3;
                    mbar_wait(mbar + ns1, ((k + 1) / 3) & 1);
                    issue_gather(ns1);
                }
                // pack slot (k + 2) % 3 held row k - 1, finished by every warp
                if (lane == 0 && r + 2 * rs < nrows)
                    issue_pack(r + 2 * rs, (k + 2) % 3);
            }
        }
        __syncwarp();
        // ---- phase 2: (block slot, own sample) register accumulation
        for (int it = lane; it < nslots * ns; it += 32) {
            const int slot = it / ns, t = t0 + (it - slot * ns);
            const int4 info = sinfo[slot];
            const int j = info.z;
            const bool bfix = info.w != 0;
            double K = 0.0, G0 = 0.0, G1 = 0.0, G2 = 0.0, D0 = 0.0, D1 = 0.0, D2 = 0.0, L = 0.0;
            for (int p = info.x; p < info.y; ++p) {
                const double2* rp = reinterpret_cast<const double2*>(rec + p * 8);
                const double2 ra = rp[0], rb = rp[1], rc = rp[2], rd = rp[3];
                const double* sp = summ + (long)__double_as_longlong(rd.y) * SI + t;
                const double gb0 = rc.x, gb1 = rc.y, gb2 = rd.x;
                K = fma(sp[0], gb0, fma(sp[SC], gb1, fma(sp[2 * SC], gb2, K)));
                const double z0 = sp[3 * SC], z1 = sp[4 * SC], z2 = sp[5 * SC];
                const double al = fma(z0, ra.x, fma(z1, ra.y, z2 * rb.x));
                G0 = fma(al, gb0, G0);
                G1 = fma(al, gb1, G1);
                G2 = fma(al, gb2, G2);
                const double alb = fma(z0, gb0, fma(z1, gb1, z2 * gb2));
                D0 = fma(ra.x, alb, D0);
                D1 = fma(ra.y, alb, D1);
                D2 = fma(rb.x, alb, D2);
                L = fma(rb.y, sp[6 * SC], L);
            }
            if (slot >= dparts || slot == 0) {
                const double2* bc = reinterpret_cast<const double2*>(blkc + j * 8);
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
                double* out = a.pvals + ((long)(k0 + j) * 8) * N + t;
                __stcs(out, K);
                __stcs(out + N, G0);
                __stcs(out + 2 * N, G1);
                __stcs(out + 3 * N, G2);
                __stcs(out + 4 * N, D0);
                __stcs(out + 5 * N, D1);
                __stcs(out + 6 * N, D2);
                __stcs(out + 7 * N, L);
            } else {
                double* o = dpart + (size_t)slot * 8 * N + t;
                o[0] = K;
                o[N] = G0;
                o[2 * N] = G1;
                o[3 * N] = G2;
                o[4 * N] = D0;
                o[5 * N] = D1;
                o[6 * N] = D2;
                o[7 * N] = L;
            }
        }
        __syncwarp();
        // ---- diagonal block: its parts summed in order (identity K on Dirichlet
        // rows, assembly.cpp:659-665), this warp's samples
        const long dblk = k0 + kdiag;
        for (int it = lane; it < 8 * ns; it += 32) {
            const int sl = it / ns, t = t0 + (it - sl * ns);
            double v = 0.0;
            for (int p = 0; p < dparts; ++p)
                v += dpart[((size_t)p * 8 + sl) * N + t];
            if (sl == 0 && afix)
                v = 1.0;
            __stcs(a.pvals + (dblk * 8 + sl) * N + t, v);
        }
        __syncwarp();
    }
    if (bad_acc)
        atomicOr(a.flag, 1);
}

// Compile-time time-sample counts (the BASELINE configs, N = 2 Nm - 1 >= 5).
#define HBGPU_WS_NC_LIST(X) X(5) X(7) X(19) X(31) X(47)
bool tangent_ws_supported(int N) {
#define HBGPU_WS_IS(n) if (N == n) return true;
    HBGPU_WS_NC_LIST(HBGPU_WS_IS)
#undef HBGPU_WS_IS
    return false;
}

template <int T>
static cudaError_t configure_ws_t(size_t bytes) {
    const int b = int(bytes < 48 * 1024 ? 48 * 1024 : bytes);
    cudaError_t e = cudaSuccess;
#define HBGPU_CFG_WS(n)                                                                                        \
    if (e == cudaSuccess)                                                                                      \
        e = cudaFuncSetAttribute(tangent_ws_kernel<0, T, n>, cudaFuncAttributeMaxDynamicSharedMemorySize, b); \
    if (e == cudaSuccess)                                                                                      \
        e = cudaFuncSetAttribute(tangent_ws_kernel<1, T, n>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    HBGPU_WS_NC_LIST(HBGPU_CFG_WS)
#undef HBGPU_CFG_WS
    return e;
}

cudaError_t configure_tangent_ws_smem(int threads, size_t bytes) {
    switch (threads) {
    case 64: return configure_ws_t<64>(bytes);
    case 128: return configure_ws_t<128>(bytes);
    case 256: return configure_ws_t<256>(bytes);
    case 512: return configure_ws_t<512>(bytes);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t tangent_ws_occupancy(int threads, int* blocks_per_sm, size_t smem) {
    switch (threads) {
    case 64: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tangent_ws_kernel<0, 64, 47>, 64, smem);
    case 128: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tangent_ws_kernel<0, 128, 47>, 128, smem);
    case 256: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tangent_ws_kernel<0, 256, 47>, 256, smem);
    case 512: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tangent_ws_kernel<0, 512, 47>, 512, smem);
    default: return cudaErrorInvalidValue;
    }
}

template <int T>
static void launch_ws_t(const TangentArgs& a, const PipeArgs& p, const double* recs, const long* rec_ptr,
                        int grid, size_t smem, cudaStream_t st) {
    switch (a.N) {
#define HBGPU_LAUNCH_WS(n)                                                                 \
    case n:                                                                                \
        if (a.tau_mode == 1)                                                               \
            tangent_ws_kernel<1, T, n><<<grid, T, smem, st>>>(a, p, recs, rec_ptr);        \
        else                                                                               \
            tangent_ws_kernel<0, T, n><<<grid, T, smem, st>>>(a, p, recs, rec_ptr);        \
        return;
        HBGPU_WS_NC_LIST(HBGPU_LAUNCH_WS)
#undef HBGPU_LAUNCH_WS
    default:
        return;
    }
}

void launch_tangent_ws(const TangentArgs& a, const PipeArgs& p, const double* recs, const long* rec_ptr,
                       int threads, int grid, size_t smem, cudaStream_t st) {
    if (p.nrows <= 0)
        return;
    note_launch();
    switch (threads) {
    case 64: launch_ws_t<64>(a, p, recs, rec_ptr, grid, smem, st); break;
    case 128: launch_ws_t<128>(a, p, recs, rec_ptr, grid, smem, st); break;
    case 256: launch_ws_t<256>(a, p, recs, rec_ptr, grid, smem, st); break;
    default: launch_ws_t<512>(a, p, recs, rec_ptr, grid, smem, st); break;
    }
}

}  // namespace hbgpu
