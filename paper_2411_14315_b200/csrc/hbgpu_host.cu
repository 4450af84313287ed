// Host runtime and C ABI of libhbgpu.so (see include/hbgpu.h).
//
// Owns the device copies of mesh, geometry, NodePattern, element incidence
// lists, colour classes and solver work buffers; orchestrates the kernels in
// hbgpu_kernels.cu on one CUDA stream.  The Newton driver mirrors
// solve_harmonic (/root/reference/proj/src/hb_solver.cpp:113-221) and the
// Krylov driver mirrors gmres_solve (src/linalg.cpp:167-293) with the
// Hessenberg / Givens bookkeeping on the host and all vector work on device.
#include "../../include/hbgpu.h"
#include "hbgpu_internal.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

using namespace hbgpu;

namespace {

thread_local std::string g_create_error;

struct Timer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double seconds() const {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
};

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t alloc(size_t count) {
        release();
        n = count;
        if (count == 0)
            return cudaSuccess;
        return cudaMalloc(reinterpret_cast<void**>(&p), sizeof(T) * count);
    }
    void release() {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

struct HostPatch {
    int kind = 0;
    std::vector<int> facets;      // 3 per facet
    std::vector<double> normals;  // 3 per facet
    std::vector<double> areas;
    double area = 0.0;
};

}  // namespace

// Test / tooling switches, read ONCE when a context is created (never on a
// hot call).  Defaults are the measured best; see DESIGN.md "Tooling switches".
struct Tooling {
    int res_tile = 0;           // HBGPU_RES_TILE: 1, 2 or 4 samples per residual tile (0 = auto)
    bool tangent_rows = false;  // HBGPU_TANGENT_KERNEL=rows: the tiled row-kernel fallback
    int tan_width = 0;          // HBGPU_TAN_WIDTH: force the tangent pipeline's CTA width
    bool gmres_host = false;    // HBGPU_GMRES_HOST: host-driven GMRES step loop
    int mv_lanes = 0;           // HBGPU_MV_LANES: 1 / 4 lanes per (row, sample) (0 = auto)
    std::string solve_progress; // HBGPU_SOLVE_PROGRESS=path: one line per Newton iteration (long solves)
    static Tooling from_env() {
        Tooling t;
        auto num = [](const char* k) { const char* v = std::getenv(k); return v ? std::atoi(v) : 0; };
        t.res_tile = num("HBGPU_RES_TILE");
        const char* tk = std::getenv("HBGPU_TANGENT_KERNEL");
        t.tangent_rows = tk && std::strcmp(tk, "rows") == 0;
        t.tan_width = num("HBGPU_TAN_WIDTH");
        t.gmres_host = std::getenv("HBGPU_GMRES_HOST") != nullptr;
        t.mv_lanes = num("HBGPU_MV_LANES");
        if (const char* sp = std::getenv("HBGPU_SOLVE_PROGRESS"))
            t.solve_progress = sp;
        return t;
    }
};

struct hbgpu_ctx {
    Tooling tool;
    // host operator of hbgpu_gmres_apply (gmres_solve(apply, ...), linalg.hpp:107-109):
    // while set, GMRES applies it through host buffers instead of the L-matvec
    hbgpu_apply_fn host_op = nullptr;
    void* host_op_user = nullptr;
    long host_n = 0;                   // vector length of the host operator
    std::vector<double> host_in, host_out;
    int nn = 0, ne = 0;
    int M = 0, N = 0;
    double period = 1.0, omega = 0.0;
    double rho = 1.06, mu = 0.04;
    int tau_mode = 0;
    double pseudo_dt = std::numeric_limits<double>::infinity();
    double pseudo_c1 = 1.5;
    int backflow_tangent = 0;
    double h_c = 0.0;

    std::vector<int> conn_h;
    std::vector<uint8_t> dir_h;
    std::vector<HostPatch> patches;
    std::vector<int> row_ptr_h, col_idx_h;
    long long nnz = 0;

    // device mesh structures
    DBuf<int4> conn;
    DBuf<double> geom;
    DBuf<uint8_t> dir;
    DBuf<int4> inc_rec;
    DBuf<int> contrib_ptr;
    DBuf<uint16_t> contrib;
    int max_inc = 0;
    // tangent rows bucketed by valence (incidences <= 24 / 32 / 48 / 64 / 96 /
    // more), so high-valence rows do not set the shared-memory size (and CTA
    // width) of every CTA
    struct TanBucket {
        DBuf<int4> desc;  // per row {A, i0, ninc, k0}, {nblk, cb, kdiag, 0}
        int count = 0, max_inc = 0, max_blk = 0, nt = 1;
        size_t smem = 0;
        // persistent row pipeline (used when its shared memory fits)
        DBuf<unsigned char> pack;
        DBuf<int> pack_ptr;
        int max_pack = 0, grid = 0, threads = 128;
        bool pipe = false;
    } tb[6];
    DBuf<double> blkc;        // per block: n-invariant tangent sums (8)
    DBuf<uint8_t> blk_order;  // per row: off-diagonal blocks by descending contribution count
    DBuf<double> tgeom;
    DBuf<int> row_ptr, col_idx, diag_blk, inc_ptr;
    DBuf<int> mv_perm;  // L-matvec row order: by descending length within 4096-row windows
    DBuf<int4> mv_rows; // {A, row_ptr[A], row_ptr[A+1], 0} in that order
    // residual element chunks
    int nchunks = 0, max_nloc = 0, res_grid = 0, res_tile = 4;
    long npairs = 0;
    DBuf<int> rpack_ptr, npart_ptr, npart;
    DBuf<unsigned char> rpack;  // chunk packs (see ResidualChunkArgs)
    int max_rpack = 0;
    DBuf<double> rpartial;


    // spectral + BCs
    DBuf<double> H;
    DBuf<double> g;
    std::vector<double> g_h;
    DBuf<double> hN;
    std::vector<double> h_h;
    std::vector<int> bc_patch;
    double beta = 0.2;
    DBuf<int> bnode, bptr, binc, fac, fbc;
    // resistance outlets (set_resistance): per patch its nodes and flux weights b
    int nres = 0;
    DBuf<int> res_ptr, res_node;
    DBuf<double> res_b, res_R;
    DBuf<double> fnormal, farea;
    int nbnodes = 0;

    // work buffers
    DBuf<double> state, r, hu, pvals, mass, mass_c, inv, y, out, x, w, z, scale, b, tmp;
    DBuf<double> V;
    DBuf<double> partial, red;
    double* h_red = nullptr;  // pinned
    size_t red_cap = 1024;
    DBuf<int> flag, ideg;
    int* h_int = nullptr;  // pinned
    // device-resident Arnoldi state of gmres_dev (see arnoldi_step_kernel)
    DBuf<double> arn;
    DBuf<int> arn_ctl;
    size_t arn_m = 0, arn_hist = 0;
    int* h_ctl = nullptr;  // pinned, 3 slots x 4
    cudaEvent_t ctl_ev[2] = {nullptr, nullptr};

    bool mass_valid = false, p_valid = false, inv_valid = false;

    // optional per-phase CUDA-event timing on the context stream
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Pair {
        int phase;
        size_t e0, e1;
    };
    std::vector<Pair> pairs;
    cudaStream_t stream = nullptr;
    // second stream: the tangent runs concurrently with the residual
    cudaStream_t stream2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::string err;

    long long state_len() const { return (long long)nn * 4 * N; }
};

#define CK(ctx, expr)                                                              \
    do {                                                                           \
        cudaError_t e_ = (expr);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            (ctx)->err = std::string(#expr) + ": " + cudaGetErrorString(e_);       \
            return e_ == cudaErrorMemoryAllocation ? HBGPU_ERR_OOM : HBGPU_ERR_CUDA; \
        }                                                                          \
    } while (0)

#define TRY(expr)            \
    do {                     \
        int s_ = (expr);     \
        if (s_ != HBGPU_OK)  \
            return s_;       \
    } while (0)

enum Phase {
    kPhResidual = 0,
    kPhResHu,
    kPhResElem,
    kPhResFinal,
    kPhTangent,
    kPhMatvec,
    kPhJacobi,
    kPhGmres,
    kPhMass,
    kPhGmDots,  // device-resident GMRES step: dot pass + its reduction
    kPhGmArnoldi,
    kPhGmUpdate,  // update pass + normalisation
    kPhGmMatvec,
    kPhCount
};

static long prof_mark(hbgpu_ctx* c) {
    if (!c->prof)
        return -1;
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess)
            return -1;
        c->ev_pool.push_back(e);
    }
    cudaEventRecord(c->ev_pool[c->ev_used], c->stream);
    return long(c->ev_used++);
}

static void prof_pair(hbgpu_ctx* c, int phase, long e0, long e1) {
    if (e0 >= 0 && e1 >= 0)
        c->pairs.push_back({phase, size_t(e0), size_t(e1)});
}

static int fail(hbgpu_ctx* c, int code, const std::string& msg) {
    c->err = msg;
    return code;
}

static int check_launch(hbgpu_ctx* c) {
    CK(c, cudaGetLastError());
    return HBGPU_OK;
}

// Singular-tau flag raised inside the element kernels -> std::domain_error.
static int check_flag(hbgpu_ctx* c) {
    CK(c, cudaMemcpyAsync(c->h_int, c->flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    const int f = c->h_int[0];
    if (f) {
        CK(c, cudaMemsetAsync(c->flag.p, 0, sizeof(int), c->stream));
        if (f & 2)
            return fail(c, HBGPU_ERR_GEOMETRY, "element has non-positive volume");
        return fail(c, HBGPU_ERR_DOMAIN,
                    "singular stabilization parameter: zero velocity with zero viscosity");
    }
    return HBGPU_OK;
}

// ---------------------------------------------------------------- host builders

// NodePattern::build semantics (linalg.cpp:10-30): element adjacency plus the
// diagonal, sorted unique columns per row.
static void build_pattern(int nn, int ne, const int* conn, std::vector<int>& row_ptr,
                          std::vector<int>& col_idx) {
    std::vector<int> cnt(size_t(nn) + 1, 0);
    for (long e = 0; e < ne; ++e)
        for (int a = 0; a < 4; ++a)
            cnt[size_t(conn[4 * e + a]) + 1] += 4;
    for (int a = 0; a < nn; ++a)
        cnt[size_t(a) + 1] += cnt[size_t(a)] + 1;
    std::vector<int> buf(static_cast<size_t>(cnt[size_t(nn)]));
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int a = 0; a < nn; ++a)
        buf[size_t(fill[size_t(a)]++)] = a;
    for (long e = 0; e < ne; ++e)
        for (int a = 0; a < 4; ++a) {
            const int A = conn[4 * e + a];
            for (int b = 0; b < 4; ++b)
                buf[size_t(fill[size_t(A)]++)] = conn[4 * e + b];
        }
    row_ptr.assign(size_t(nn) + 1, 0);
    col_idx.clear();
    col_idx.reserve(buf.size() / 3);
    for (int a = 0; a < nn; ++a) {
        auto b0 = buf.begin() + cnt[size_t(a)], b1 = buf.begin() + cnt[size_t(a) + 1];
        std::sort(b0, b1);
        auto last = std::unique(b0, b1);
        col_idx.insert(col_idx.end(), b0, last);
        row_ptr[size_t(a) + 1] = int(col_idx.size());
    }
}

static int upload_all(hbgpu_ctx* c, const hbgpu_mesh_desc* d) {
    const int nn = c->nn, ne = c->ne;
    cudaStream_t st = c->stream;
    CK(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_red), sizeof(double) * 1024));
    CK(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_int), sizeof(int) * 16));
    CK(c, c->conn.alloc(size_t(ne)));
    CK(c, cudaMemcpyAsync(c->conn.p, d->conn, sizeof(int4) * size_t(ne), cudaMemcpyHostToDevice, st));
    CK(c, c->dir.alloc(size_t(nn)));
    CK(c, cudaMemcpyAsync(c->dir.p, c->dir_h.data(), size_t(nn), cudaMemcpyHostToDevice, st));
    CK(c, c->flag.alloc(1));
    CK(c, c->ideg.alloc(1));
    CK(c, cudaMemsetAsync(c->flag.p, 0, sizeof(int), st));
    CK(c, c->geom.alloc(size_t(ne) * 22));
    if (d->geometry) {
        CK(c, cudaMemcpyAsync(c->geom.p, d->geometry, sizeof(double) * 22 * size_t(ne),
                              cudaMemcpyHostToDevice, st));
    } else {
        DBuf<double> xyz;
        CK(c, xyz.alloc(size_t(nn) * 3));
        CK(c, cudaMemcpyAsync(xyz.p, d->xyz, sizeof(double) * 3 * size_t(nn),
                              cudaMemcpyHostToDevice, st));
        launch_geometry(xyz.p, c->conn.p, ne, c->geom.p, c->flag.p, st);
        TRY(check_launch(c));
        CK(c, cudaStreamSynchronize(st));
        xyz.release();
        TRY(check_flag(c));
    }

    // pattern + per-row diagonal
    build_pattern(nn, ne, d->conn, c->row_ptr_h, c->col_idx_h);
    c->nnz = (long long)c->col_idx_h.size();
    std::vector<int> diag(static_cast<size_t>(nn));
    for (int A = 0; A < nn; ++A) {
        const int* b0 = c->col_idx_h.data() + c->row_ptr_h[size_t(A)];
        const int* b1 = c->col_idx_h.data() + c->row_ptr_h[size_t(A) + 1];
        diag[size_t(A)] = int(std::lower_bound(b0, b1, A) - c->col_idx_h.data());
    }
    CK(c, c->row_ptr.alloc(size_t(nn) + 1));
    CK(c, c->col_idx.alloc(size_t(c->nnz)));
    CK(c, c->diag_blk.alloc(size_t(nn)));
    CK(c, cudaMemcpyAsync(c->row_ptr.p, c->row_ptr_h.data(), sizeof(int) * (size_t(nn) + 1),
                          cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->col_idx.p, c->col_idx_h.data(), sizeof(int) * size_t(c->nnz),
                          cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->diag_blk.p, diag.data(), sizeof(int) * size_t(nn),
                          cudaMemcpyHostToDevice, st));
    {
        // L-matvec row order: a CTA's rows finish together when their block
        // counts match, so rows are stably sorted by descending length inside
        // windows of 4096 consecutive rows (y stays L2-local per window)
        std::vector<int> perm(static_cast<size_t>(nn));
        for (int A = 0; A < nn; ++A)
            perm[size_t(A)] = A;
        const int* rp = c->row_ptr_h.data();
        const int win = 4096;
        for (int w0 = 0; w0 < nn; w0 += win) {
            const int w1 = std::min(nn, w0 + win);
            std::stable_sort(perm.begin() + w0, perm.begin() + w1, [rp](int x, int y) {
                return rp[x + 1] - rp[x] > rp[y + 1] - rp[y];
            });
        }
        CK(c, c->mv_perm.alloc(size_t(nn)));
        CK(c, cudaMemcpyAsync(c->mv_perm.p, perm.data(), sizeof(int) * size_t(nn), cudaMemcpyHostToDevice, st));
        std::vector<int4> rows(static_cast<size_t>(nn));
        for (int q = 0; q < nn; ++q) {
            const int A = perm[size_t(q)];
            rows[size_t(q)] = make_int4(A, rp[A], rp[A + 1], 0);
        }
        CK(c, c->mv_rows.alloc(size_t(nn)));
        CK(c, cudaMemcpyAsync(c->mv_rows.p, rows.data(), sizeof(int4) * size_t(nn), cudaMemcpyHostToDevice, st));
        CK(c, cudaStreamSynchronize(st));
    }

    // element incidences per row, element order; local block offsets
    std::vector<int> iptr(size_t(nn) + 1, 0);
    for (long e = 0; e < ne; ++e)
        for (int a = 0; a < 4; ++a)
            iptr[size_t(d->conn[4 * e + a]) + 1] += 1;
    for (int A = 0; A < nn; ++A)
        iptr[size_t(A) + 1] += iptr[size_t(A)];
    // record per incidence: conn[4] | {e | a<<30, 4 x u8 block offsets, Dirichlet mask, 0}
    std::vector<int4> irec(size_t(8) * size_t(ne));
    std::vector<int> fill(iptr.begin(), iptr.end() - 1);
    for (long e = 0; e < ne; ++e) {
        int m = 0;
        for (int b = 0; b < 4; ++b)
            m |= (c->dir_h[size_t(d->conn[4 * e + b])] ? 1 : 0) << b;
        for (int a = 0; a < 4; ++a) {
            const int A = d->conn[4 * e + a];
            const int* r0 = c->col_idx_h.data() + c->row_ptr_h[size_t(A)];
            const int* r1 = c->col_idx_h.data() + c->row_ptr_h[size_t(A) + 1];
            uint32_t cols = 0;
            for (int b = 0; b < 4; ++b) {
                const long off = std::lower_bound(r0, r1, d->conn[4 * e + b]) - r0;
                if (off > 255)
                    return fail(c, HBGPU_ERR_INVALID, "node degree above 255 blocks per row");
                cols |= uint32_t(off) << (8 * b);
            }
            const int slot = fill[size_t(A)]++;
            irec[2 * size_t(slot)] = make_int4(d->conn[4 * e], d->conn[4 * e + 1],
                                               d->conn[4 * e + 2], d->conn[4 * e + 3]);
            irec[2 * size_t(slot) + 1] =
                make_int4(int(uint32_t(e) | (uint32_t(a) << 30)), int(cols), m, 0);
        }
    }
    CK(c, c->inc_ptr.alloc(size_t(nn) + 1));
    CK(c, c->inc_rec.alloc(irec.size()));
    CK(c, cudaMemcpyAsync(c->inc_ptr.p, iptr.data(), sizeof(int) * iptr.size(),
                          cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->inc_rec.p, irec.data(), sizeof(int4) * irec.size(),
                          cudaMemcpyHostToDevice, st));
    CK(c, c->tgeom.alloc(size_t(ne) * kTGeo));
    launch_tangent_geometry(c->geom.p, ne, c->tgeom.p, st);
    TRY(check_launch(c));
    // per block: its (incidence-in-row, b) contributions in element order
    {
        std::vector<int> cptr(size_t(c->nnz) + 1, 0);
        int max_inc = 0;
        for (int A = 0; A < nn; ++A) {
            max_inc = std::max(max_inc, iptr[size_t(A) + 1] - iptr[size_t(A)]);
            for (int s = iptr[size_t(A)]; s < iptr[size_t(A) + 1]; ++s) {
                const uint32_t cols = uint32_t(irec[2 * size_t(s) + 1].y);
                for (int b = 0; b < 4; ++b)
                    cptr[size_t(c->row_ptr_h[size_t(A)] + int((cols >> (8 * b)) & 0xFF)) + 1] += 1;
            }
        }
        if (max_inc >= 16384)
            return fail(c, HBGPU_ERR_INVALID, "node with more than 16383 elements");
        for (long k = 0; k < c->nnz; ++k)
            cptr[size_t(k) + 1] += cptr[size_t(k)];
        std::vector<uint16_t> contrib(static_cast<size_t>(cptr[size_t(c->nnz)]));
        std::vector<int> cf(cptr.begin(), cptr.end() - 1);
        for (int A = 0; A < nn; ++A)
            for (int s = iptr[size_t(A)]; s < iptr[size_t(A) + 1]; ++s) {
                const uint32_t cols = uint32_t(irec[2 * size_t(s) + 1].y);
                const int i = s - iptr[size_t(A)];
                for (int b = 0; b < 4; ++b) {
                    const int k = c->row_ptr_h[size_t(A)] + int((cols >> (8 * b)) & 0xFF);
                    contrib[size_t(cf[size_t(k)]++)] = uint16_t((i << 2) | b);
                }
            }
        c->max_inc = max_inc;
        // off-diagonal blocks of each row, longest contribution list first
        std::vector<uint8_t> order(size_t(c->nnz), 0);
        for (int A = 0; A < nn; ++A) {
            const int k0 = c->row_ptr_h[size_t(A)], nb = c->row_ptr_h[size_t(A) + 1] - k0;
            std::vector<int> js;
            for (int j = 0; j < nb; ++j)
                if (c->col_idx_h[size_t(k0 + j)] != A)
                    js.push_back(j);
            std::stable_sort(js.begin(), js.end(), [&](int x, int y) {
                return cptr[size_t(k0 + x) + 1] - cptr[size_t(k0 + x)] >
                       cptr[size_t(k0 + y) + 1] - cptr[size_t(k0 + y)];
            });
            for (size_t s2 = 0; s2 < js.size(); ++s2)
                order[size_t(k0) + s2] = uint8_t(js[s2]);
        }
        std::vector<int> brows[6];
        for (int A = 0; A < nn; ++A) {
            const int ni = iptr[size_t(A) + 1] - iptr[size_t(A)];
            const int bk = ni <= 24 ? 0 : ni <= 32 ? 1 : ni <= 48 ? 2 : ni <= 64 ? 3 : ni <= 96 ? 4 : 5;
            brows[bk].push_back(A);
            c->tb[bk].max_inc = std::max(c->tb[bk].max_inc, ni);
            c->tb[bk].max_blk = std::max(c->tb[bk].max_blk,
                                         c->row_ptr_h[size_t(A) + 1] - c->row_ptr_h[size_t(A)]);
        }
        for (int bk = 0; bk < 6; ++bk) {
            c->tb[bk].count = int(brows[bk].size());
            if (!c->tb[bk].count)
                continue;
            std::vector<int4> desc;
            for (int A : brows[bk]) {
                const int k0 = c->row_ptr_h[size_t(A)];
                desc.push_back(make_int4(A, iptr[size_t(A)], iptr[size_t(A) + 1] - iptr[size_t(A)], k0));
                desc.push_back(make_int4(c->row_ptr_h[size_t(A) + 1] - k0, cptr[size_t(k0)],
                                         diag[size_t(A)] - k0, 0));
            }
            CK(c, c->tb[bk].desc.alloc(desc.size()));
            CK(c, cudaMemcpyAsync(c->tb[bk].desc.p, desc.data(), sizeof(int4) * desc.size(),
                                  cudaMemcpyHostToDevice, st));
            // row packs for the persistent pipeline
            std::vector<int> pptr{0};
            for (int A : brows[bk]) {
                const int ni = iptr[size_t(A) + 1] - iptr[size_t(A)];
                const int nb = c->row_ptr_h[size_t(A) + 1] - c->row_ptr_h[size_t(A)];
                const int bytes = int(tangent_pack_bytes(ni, nb));
                c->tb[bk].max_pack = std::max(c->tb[bk].max_pack, bytes);
                pptr.push_back(pptr.back() + bytes / 16);
            }
            std::vector<unsigned char> pk(size_t(pptr.back()) * 16);
            std::vector<int2> incl;
            std::vector<int> rcptr;
            for (size_t r = 0; r < brows[bk].size(); ++r) {
                const int A = brows[bk][r];
                const int k0 = c->row_ptr_h[size_t(A)];
                const int nb = c->row_ptr_h[size_t(A) + 1] - k0;
                const int ni = iptr[size_t(A) + 1] - iptr[size_t(A)];
                incl.resize(size_t(ni));
                for (int i = 0; i < ni; ++i) {
                    const int4 r1 = irec[2 * size_t(iptr[size_t(A)] + i) + 1];
                    incl[size_t(i)] = make_int2(r1.x, r1.y);
                }
                rcptr.resize(size_t(nb) + 1);
                for (int j = 0; j <= nb; ++j)
                    rcptr[size_t(j)] = cptr[size_t(k0 + j)] - cptr[size_t(k0)];
                tangent_pack_write(pk.data() + size_t(pptr[r]) * 16, A, k0, ni, nb, diag[size_t(A)] - k0,
                                   c->col_idx_h.data() + k0, incl.data(),
                                   contrib.data() + cptr[size_t(k0)], rcptr.data(), order.data() + k0);
            }
            CK(c, c->tb[bk].pack.alloc(pk.size()));
            CK(c, c->tb[bk].pack_ptr.alloc(pptr.size()));
            CK(c, cudaMemcpyAsync(c->tb[bk].pack.p, pk.data(), pk.size(), cudaMemcpyHostToDevice, st));
            CK(c, cudaMemcpyAsync(c->tb[bk].pack_ptr.p, pptr.data(), sizeof(int) * pptr.size(),
                                  cudaMemcpyHostToDevice, st));
        }
        CK(c, c->contrib_ptr.alloc(cptr.size()));
        CK(c, c->contrib.alloc(contrib.size()));
        CK(c, cudaMemcpyAsync(c->contrib_ptr.p, cptr.data(), sizeof(int) * cptr.size(),
                              cudaMemcpyHostToDevice, st));
        CK(c, cudaMemcpyAsync(c->contrib.p, contrib.data(), sizeof(uint16_t) * contrib.size(),
                              cudaMemcpyHostToDevice, st));
        CK(c, c->blk_order.alloc(order.size()));
        CK(c, cudaMemcpyAsync(c->blk_order.p, order.data(), order.size(), cudaMemcpyHostToDevice, st));
        CK(c, c->blkc.alloc(size_t(c->nnz) * 8));
        launch_tangent_blockconst(c->tgeom.p, c->row_ptr.p, c->inc_ptr.p, c->inc_rec.p,
                                  c->contrib_ptr.p, c->contrib.p, nn, c->blkc.p, st);
        for (auto& b : c->tb)
            launch_tangent_pack_refresh(b.pack.p, b.pack_ptr.p, b.count, c->dir.p, c->blkc.p, st);
        TRY(check_launch(c));
        CK(c, cudaStreamSynchronize(st));
    }

    // element chunks of kChunkElems consecutive elements: distinct nodes,
    // chunk-local connectivity, per (chunk, node) slot lists in element order,
    // and per node the (chunk, node) records in chunk order
    const int CE = kChunkElems;
    const int nch = (ne + CE - 1) / CE;
    std::vector<int> cnodes, npp(size_t(nn) + 1, 0), npl, rpp{0};
    std::vector<unsigned char> rpk;
    int maxnloc = 0, maxpk = 0;
    for (int ch = 0; ch < nch; ++ch) {
        const long e0 = long(ch) * CE, e1 = std::min<long>(ne, e0 + CE);
        const int ecount = int(e1 - e0);
        std::vector<int> loc;
        for (long e = e0; e < e1; ++e)
            for (int a = 0; a < 4; ++a)
                loc.push_back(d->conn[4 * e + a]);
        std::sort(loc.begin(), loc.end());
        loc.erase(std::unique(loc.begin(), loc.end()), loc.end());
        if (loc.size() > 255)
            return fail(c, HBGPU_ERR_INVALID, "element chunk with more than 255 nodes");
        const int nloc = int(loc.size());
        maxnloc = std::max(maxnloc, nloc);
        std::vector<std::vector<uint8_t>> inc(loc.size());
        std::vector<uint32_t> lconn(size_t(ecount), 0);
        for (long e = e0; e < e1; ++e) {
            uint32_t pk = 0;
            for (int a = 0; a < 4; ++a) {
                const int ln = int(std::lower_bound(loc.begin(), loc.end(), d->conn[4 * e + a]) - loc.begin());
                pk |= uint32_t(ln) << (8 * a);
                inc[size_t(ln)].push_back(uint8_t((e - e0) * 4 + a));
            }
            lconn[size_t(e - e0)] = pk;
        }
        // slot lists as offsets into the kernel's per-element slot array:
        // element stride 29T (bank padding), output-group stride 7T
        std::vector<int> sptr{0};
        std::vector<uint16_t> soff;
        const int nb = int(cnodes.size());
        for (int ln = 0; ln < nloc; ++ln) {
            cnodes.push_back(loc[size_t(ln)]);
            for (uint8_t sl : inc[size_t(ln)])
                soff.push_back(uint16_t((sl >> 2) * 29 + (sl & 3) * 7));
            sptr.push_back(int(soff.size()));
            npp[size_t(loc[size_t(ln)]) + 1] += 1;
        }
        const int bytes = int(residual_pack_bytes(nloc, ecount));
        maxpk = std::max(maxpk, bytes);
        rpk.resize(rpk.size() + size_t(bytes));
        residual_pack_write(rpk.data() + rpk.size() - size_t(bytes), nloc, ecount, nb, loc.data(),
                            sptr.data(), soff.data(), lconn.data());
        rpp.push_back(rpp.back() + bytes / 16);
    }
    for (int A = 0; A < nn; ++A)
        npp[size_t(A) + 1] += npp[size_t(A)];
    npl.assign(cnodes.size(), 0);
    {
        std::vector<int> f(npp.begin(), npp.end() - 1);
        for (size_t p = 0; p < cnodes.size(); ++p)
            npl[size_t(f[size_t(cnodes[p])]++)] = int(p);
    }
    c->nchunks = nch;
    c->max_nloc = maxnloc;
    c->max_rpack = maxpk;
    c->npairs = long(cnodes.size());
    CK(c, c->rpack.alloc(rpk.size()));
    CK(c, c->rpack_ptr.alloc(rpp.size()));
    CK(c, c->npart_ptr.alloc(npp.size()));
    CK(c, c->npart.alloc(npl.size()));
    CK(c, cudaMemcpyAsync(c->rpack.p, rpk.data(), rpk.size(), cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->rpack_ptr.p, rpp.data(), sizeof(int) * rpp.size(), cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->npart_ptr.p, npp.data(), sizeof(int) * npp.size(), cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->npart.p, npl.data(), sizeof(int) * npl.size(), cudaMemcpyHostToDevice, st));
    CK(c, cudaStreamSynchronize(st));

    CK(c, c->partial.alloc(size_t(kRedBlocks) * 1024));
    CK(c, c->red.alloc(1024));
    CK(c, cudaStreamSynchronize(st));
    return HBGPU_OK;
}

// L-matvec CTA: MV_CTA_THREADS / N rows of N (row, sample) threads.  512:
// config 4 (N = 47) 8.29 -> 7.89 ms, config 1 (N = 19) 0.211 -> 0.196 ms
// against 256; 128 and a 4-block unroll were slower (profiles/r2i_kb_mv.jsonl)
#ifndef MV_CTA_THREADS
#define MV_CTA_THREADS 512
#endif
static int rows_per_matvec_cta(int N) { return std::max(1, MV_CTA_THREADS / N); }

// ---------------------------------------------------------------- operations

static int residual_dev(hbgpu_ctx* c, const double* d_state, double* d_r) {
    const int N = c->N;
    cudaStream_t st = c->stream;
    const long p0 = prof_mark(c);
    // nodal H*u at every node, Dirichlet ones included (assembly.cpp:453-463)
    if (N > 1)
        launch_apply_h_series(c->H.p, N, d_state, 4 * N, c->hu.p, 3 * N, c->nn, st);
    else
        CK(c, cudaMemsetAsync(c->hu.p, 0, sizeof(double) * size_t(c->nn) * 3, st));
    const long p1 = prof_mark(c);
    ResidualChunkArgs ca;
    ca.tgeom = c->tgeom.p;
    ca.state = d_state;
    ca.hu = c->hu.p;
    ca.rpack = c->rpack.p;
    ca.rpack_ptr = c->rpack_ptr.p;
    ca.max_rpack = c->max_rpack;
    ca.partial = c->rpartial.p;
    ca.ne = c->ne;
    ca.N = N;
    ca.max_nloc = c->max_nloc;
    ca.nchunks = c->nchunks;
    ca.npairs = c->npairs;
    ca.rho = c->rho;
    ca.mu = c->mu;
    ca.nu = c->mu / c->rho;
    ca.tau_mode = c->tau_mode;
    ca.flag = c->flag.p;
    launch_residual_chunks(ca, c->res_grid, c->res_tile, st);
    const long p2 = prof_mark(c);
    launch_residual_nodes(c->H.p, N, c->nn, c->npart_ptr.p, c->npart.p, c->rpartial.p, c->dir.p,
                          d_r, c->res_tile, c->npairs, st);
    if (c->nbnodes > 0) {
        BoundaryArgs b;
        b.bnode = c->bnode.p;
        b.bptr = c->bptr.p;
        b.binc = c->binc.p;
        b.fac = c->fac.p;
        b.fnormal = c->fnormal.p;
        b.farea = c->farea.p;
        b.fbc = c->fbc.p;
        b.h = c->hN.p;
        b.dir = c->dir.p;
        b.state = d_state;
        b.r = d_r;
        b.nbnodes = c->nbnodes;
        b.N = N;
        b.rho = c->rho;
        b.beta = c->beta;
        launch_boundary(b, st);
    }
    launch_resistance(c->res_ptr.p, c->res_node.p, c->res_b.p, c->res_R.p, c->nres, c->dir.p, N, d_state, d_r,
                      nullptr, 0, nullptr, st);
    const long p3 = prof_mark(c);
    prof_pair(c, kPhResidual, p0, p3);
    prof_pair(c, kPhResHu, p0, p1);
    prof_pair(c, kPhResElem, p1, p2);
    prof_pair(c, kPhResFinal, p2, p3);
    return check_launch(c);
}

static BoundaryArgs boundary_args(hbgpu_ctx* c, const double* d_state, double* d_r) {
    BoundaryArgs b;
    b.bnode = c->bnode.p;
    b.bptr = c->bptr.p;
    b.binc = c->binc.p;
    b.fac = c->fac.p;
    b.fnormal = c->fnormal.p;
    b.farea = c->farea.p;
    b.fbc = c->fbc.p;
    b.h = c->hN.p;
    b.dir = c->dir.p;
    b.state = d_state;
    b.r = d_r;
    b.nbnodes = c->nbnodes;
    b.N = c->N;
    b.rho = c->rho;
    b.beta = c->beta;
    return b;
}

static int tangent_dev(hbgpu_ctx* c, const double* d_state) {
    TangentArgs a;
    a.tgeom = c->tgeom.p;
    a.state = d_state;
    a.dir = c->dir.p;
    a.row_ptr = c->row_ptr.p;
    a.inc_ptr = c->inc_ptr.p;
    a.inc_rec = c->inc_rec.p;
    a.pvals = c->pvals.p;
    a.N = c->N;
    a.rho = c->rho;
    a.mu = c->mu;
    a.nu = c->mu / c->rho;
    const bool pseudo = std::isfinite(c->pseudo_dt);
    a.pseudo_c = pseudo ? c->pseudo_c1 * c->rho / c->pseudo_dt : 0.0;
    a.tau_mode = c->tau_mode;
    a.flag = c->flag.p;
    const long p0 = prof_mark(c);
    a.col_idx = c->col_idx.p;
    a.diag_blk = c->diag_blk.p;
    a.contrib_ptr = c->contrib_ptr.p;
    a.contrib = c->contrib.p;
    a.blkc = c->blkc.p;
    a.blk_order = c->blk_order.p;

    for (const auto& b : c->tb) {
        if (!b.count)
            continue;
        a.rowdesc = b.desc.p;
        a.max_inc = b.max_inc;
        a.max_blk = b.max_blk;
        a.NT = b.nt;
        if (b.pipe) {
            PipeArgs pa;
            pa.pack = b.pack.p;
            pa.pack_ptr = b.pack_ptr.p;
            pa.nrows = b.count;
            pa.max_pack = b.max_pack;
            launch_tangent_pipe(a, pa, b.threads, b.grid, b.smem, c->stream);
        } else {
            launch_tangent_row(a, b.count, b.smem, c->stream);
        }
    }
    if (c->backflow_tangent && c->nbnodes > 0)
        launch_backflow_tangent(boundary_args(c, d_state, nullptr), c->row_ptr.p, c->col_idx.p,
                                c->pvals.p, c->stream);
    prof_pair(c, kPhTangent, p0, prof_mark(c));
    c->p_valid = true;
    c->inv_valid = false;
    return check_launch(c);
}

static int mass_dev(hbgpu_ctx* c) {
    const long p0 = prof_mark(c);
    launch_mass_rows(c->geom.p, c->row_ptr.p, c->inc_ptr.p, c->inc_rec.p, c->rho, c->mass.p,
                     c->nn, c->stream);
    launch_mask_mass(c->mass.p, c->row_ptr.p, c->col_idx.p, c->dir.p, c->nn, c->mass_c.p,
                     c->stream);
    prof_pair(c, kPhMass, p0, prof_mark(c));
    c->mass_valid = true;
    return check_launch(c);
}

static int matvec_dev(hbgpu_ctx* c, const double* d_y, double* d_out, const double* d_scale,
                      bool with_c, const double* d_scale_out = nullptr, const int* d_skip = nullptr) {
    if (!c->p_valid)
        return fail(c, HBGPU_ERR_INVALID, "matvec before assemble_tangent / set_pvals");
    if (with_c && c->N > 1 && !c->mass_valid)
        TRY(mass_dev(c));
    MatvecArgs a;
    a.row_ptr = c->row_ptr.p;
    a.col_idx = c->col_idx.p;
    a.vals = c->pvals.p;
    a.mass = c->mass_c.p;
    a.dir = c->dir.p;
    a.H = c->H.p;
    a.y = d_y;
    a.out = d_out;
    a.scale = d_scale;
    if (d_scale)
        return fail(c, HBGPU_ERR_INVALID, "input-scaled matvec is not supported (scale z on the host side)");
    a.scale_out = d_scale_out;
    a.perm = c->mv_perm.p;
    a.rows = c->mv_rows.p;
    a.skip = d_skip;
    a.lanes = c->tool.mv_lanes;
    a.nn = c->nn;
    a.N = c->N;
    a.rows_per_cta = rows_per_matvec_cta(c->N);
    a.with_c = (with_c && c->N > 1) ? 1 : 0;
    const long p0 = prof_mark(c);
    launch_lmatvec(a, c->stream);
    if (with_c)  // resistance outlets belong to the tangent operator, not to P
        launch_resistance(c->res_ptr.p, c->res_node.p, c->res_b.p, c->res_R.p, c->nres, c->dir.p, c->N, d_y, d_out,
                          d_scale_out, 1, d_skip, c->stream);
    prof_pair(c, kPhMatvec, p0, prof_mark(c));
    return check_launch(c);
}

static int jacobi_dev(hbgpu_ctx* c, int* degenerate) {
    if (!c->p_valid)
        return fail(c, HBGPU_ERR_INVALID, "jacobi before assemble_tangent / set_pvals");
    CK(c, cudaMemsetAsync(c->ideg.p, 0, sizeof(int), c->stream));
    const long p0 = prof_mark(c);
    launch_jacobi(c->pvals.p, c->diag_blk.p, c->nn, c->N, c->inv.p, c->ideg.p, c->stream);
    prof_pair(c, kPhJacobi, p0, prof_mark(c));
    TRY(check_launch(c));
    CK(c, cudaMemcpyAsync(c->h_int + 1, c->ideg.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (degenerate)
        *degenerate = c->h_int[1];
    c->inv_valid = true;
    return HBGPU_OK;
}

// <a,b> for vectors already on device; deterministic.  Result on host.
static int dot_dev(hbgpu_ctx* c, const double* a, const double* b, long n, double* out,
                   bool take_sqrt) {
    launch_multidot(a, 0, 1, b, n, c->partial.p, c->stream);
    launch_reduce_partials(c->partial.p, 1, c->red.p, take_sqrt ? 1 : 0, c->stream);
    TRY(check_launch(c));
    CK(c, cudaMemcpyAsync(c->h_red, c->red.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    *out = c->h_red[0];
    return HBGPU_OK;
}

static int ensure_basis(hbgpu_ctx* c) {
    if (c->N <= 0)
        return fail(c, HBGPU_ERR_INVALID, "spectral basis not set (hbgpu_set_basis)");
    return HBGPU_OK;
}

// gmres_solve (linalg.cpp:167-293): split Jacobi scaling, restarted Arnoldi,
// Givens rotations, true residual recompute per cycle, stagnation when a
// cycle does not decrease it.  Orthogonalisation: classical Gram-Schmidt with
// delayed re-orthogonalisation (DCGS2): step j applies the operator to the
// tentative vector u_j, and ONE pass over V_0..V_{j-1} yields both the
// re-orthogonalisation coefficients of u_j (a = Q^T u_j) and the projections
// of w = A u_j (b = Q^T w); a second pass writes q_j = (u_j - Q a)/rho and
// the projected w.  Two passes over the basis per step instead of the four of
// CGS2, one host synchronisation, MGS-level orthogonality.  Because A u_j and
// A q_j differ, column j is derived from the Arnoldi relation A Q_j = Q_{j+1} H_j:
//   rho = sqrt(<u,u> - |a|^2),  c = [b ; (<u,w> - a.b)/rho],
//   h_{:,j} = (c - H_j a)/rho,  w' = (w - Q_{j+1} c)/rho,
// and column j-1 is finalised with the re-orthogonalisation of u_j:
//   h_{0:j,j-1} += h_{j,j-1} a,  h_{j,j-1} *= rho.
// Column j-1 is therefore final (Givens, estimate, convergence test) one step
// after its vector was produced; the reference's iteration count, history and
// restart semantics are kept per finalised column.
static int gmres_dev(hbgpu_ctx* c, const double* d_rhs, const double* d_inv,
                     const hbgpu_krylov_cfg* kc, double* d_x, hbgpu_krylov_result* res,
                     double* history, int hcap) {
    cudaStream_t st = c->stream;
    const long n = c->host_op ? c->host_n : long(c->state_len());
    const int m = std::max(1, kc->restart);
    // the operator: out = [S] A in (S: the split Jacobi scaling, d_scale_out)
    auto apply_op = [&](const double* d_in, double* d_out, const double* d_scale_out) -> int {
        if (!c->host_op)
            return matvec_dev(c, d_in, d_out, nullptr, true, d_scale_out);
        CK(c, cudaMemcpyAsync(c->host_in.data(), d_in, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, st));
        CK(c, cudaStreamSynchronize(st));
        c->host_op(c->host_op_user, c->host_in.data(), c->host_out.data());
        CK(c, cudaMemcpyAsync(d_out, c->host_out.data(), sizeof(double) * size_t(n), cudaMemcpyHostToDevice, st));
        if (d_scale_out)
            launch_mul(d_scale_out, d_out, d_out, n, st);
        return check_launch(c);
    };
    res->iterations = 0;
    res->relative_residual = 1.0;
    res->status = 0;
    res->history_len = 0;
    res->reorthogonalizations = 0;
    auto push_hist = [&](double v) {
        if (history && res->history_len < hcap)
            history[res->history_len] = v;
        res->history_len += (history && res->history_len < hcap) ? 1 : 0;
    };
    // basis capacity in doubles (the vector length differs between the
    // L-matvec and a host operator of hbgpu_gmres_apply)
    if (c->V.n < (size_t(m) + 1) * size_t(n))
        CK(c, c->V.alloc((size_t(m) + 1) * size_t(n)));
    // scratch: red[0, 2m+4) dot results | [2m+4, 4m+8) update coefficients | [4m+8] |w'|
    const size_t need = 4 * size_t(m) + 16;
    if (c->red_cap < need) {
        CK(c, c->red.alloc(need));
        CK(c, c->partial.alloc((2 * size_t(m) + 16) * kRedBlocks));
        if (c->h_red)
            cudaFreeHost(c->h_red);
        c->h_red = nullptr;
        CK(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_red), sizeof(double) * need));
        c->red_cap = need;
    }
    // HBGPU_GMRES_HOST=1 (or a restart too long for the Arnoldi kernel's shared
    // memory, m > ~700): the host-driven step loop, one synchronisation per
    // step; else the device-resident cycle
    const bool devloop = !c->tool.gmres_host && !c->host_op && arnoldi_step_smem(m) <= 200 * 1024;
    ArnoldiDev ad{};
    if (devloop) {
        const size_t hsz = size_t(m + 2) * size_t(m + 1);
        const size_t hist = size_t(std::max(kc->max_iters, 0)) + 2;
        if (c->arn_m < size_t(m) || c->arn_hist < hist) {
            CK(c, c->arn.alloc(2 * hsz + 3 * (size_t(m) + 2) + hist));
            c->arn_m = size_t(m);
            c->arn_hist = hist;
        }
        if (!c->arn_ctl.p) {
            CK(c, c->arn_ctl.alloc(4));
            CK(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_ctl), sizeof(int) * 12));
            for (auto& e : c->ctl_ev)
                CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        ad.Hm = c->arn.p;
        ad.R = ad.Hm + hsz;
        ad.cs = ad.R + hsz;
        ad.sn = ad.cs + (m + 2);
        ad.gv = ad.sn + (m + 2);
        ad.hist = ad.gv + (m + 2);
        ad.ctl = c->arn_ctl.p;
        ad.m = m;
        ad.hcap = int(std::min<size_t>(hist, size_t(std::max(hcap, 0))));
        if (arnoldi_step_smem(m) > 48 * 1024)
            CK(c, configure_arnoldi_smem(m));
    }
    // device history (indexed by iteration) -> caller's buffer, at every exit
    auto pull_hist = [&]() -> int {
        if (!devloop || !history || hcap <= 1 || res->iterations <= 0)
            return HBGPU_OK;
        const int cnt = std::min(res->iterations + 1, std::min(hcap, ad.hcap));
        if (cnt > 1)
            CK(c, cudaMemcpy(history + 1, ad.hist + 1, sizeof(double) * size_t(cnt - 1), cudaMemcpyDeviceToHost));
        res->history_len = cnt;
        return HBGPU_OK;
    };
    double* V = c->V.p;
    const size_t o_coef = 2 * size_t(m) + 4, o_norm = 4 * size_t(m) + 8;
    double* d_norm = c->red.p + o_norm;
    double* d_coef = c->red.p + o_coef;
    double* h_coef = c->h_red + o_coef;
    launch_sqrt_abs(d_inv, c->scale.p, n, st);
    launch_mul(c->scale.p, d_rhs, c->b.p, n, st);
    CK(c, cudaMemsetAsync(d_x, 0, sizeof(double) * size_t(n), st));
    double bnorm = 0.0;
    TRY(dot_dev(c, c->b.p, c->b.p, n, &bnorm, true));
    if (bnorm == 0.0) {
        res->relative_residual = 0.0;
        return HBGPU_OK;
    }
    std::vector<double> Hm(static_cast<size_t>((m + 2) * (m + 1))), R(static_cast<size_t>((m + 2) * (m + 1))),
        cs(static_cast<size_t>(m + 1)), sn(static_cast<size_t>(m + 1)), gv(static_cast<size_t>(m + 2)),
        yv(static_cast<size_t>(m + 1)), av(static_cast<size_t>(m + 1));
    // H: the (unrotated) Hessenberg matrix of the Arnoldi relation;
    // R: its Givens-rotated copy (columns rotated once final)
    auto HH = [&](int i, int j) -> double& { return Hm[size_t(j) * size_t(m + 2) + size_t(i)]; };
    auto RR = [&](int i, int j) -> double& { return R[size_t(j) * size_t(m + 2) + size_t(i)]; };
    double rnorm = bnorm;
    const double* rsrc = c->b.p;
    push_hist(1.0);
    while (res->iterations < kc->max_iters) {
        const double cycle_start = rnorm;
        std::fill(Hm.begin(), Hm.end(), 0.0);
        std::fill(R.begin(), R.end(), 0.0);
        std::fill(gv.begin(), gv.end(), 0.0);
        gv[0] = rnorm;
        if (!devloop) {
            c->h_red[0] = rnorm;
            CK(c, cudaMemcpyAsync(c->red.p, c->h_red, sizeof(double), cudaMemcpyHostToDevice, st));
            // V_0 = r/|r| (exactly normalised), z = S V_0
            launch_normalize(rsrc, c->red.p, V, n, st, c->scale.p, c->z.p);
        }
        int ncols = 0;  // finalised columns of this cycle
        if (devloop) {
            // Device-resident cycle: the dense Arnoldi/Givens work of each step
            // runs in arnoldi_step_kernel, so steps are enqueued in batches of
            // kBatch with no host round trip; the host polls the stop flag one
            // batch behind (steps enqueued past a stop return at once).
            // steps per host poll: 4 / 8 / 16 / 32 measured equal on the config-0
            // solve (0.677 / 0.670 / 0.670 / 0.675 s): the cycle is kernel-bound
            constexpr int kBatch = 8;
            const int it0 = res->iterations;
            launch_arnoldi_init(ad, rnorm, it0, res->reorthogonalizations, c->red.p, st);
            launch_normalize(rsrc, c->red.p, V, n, st, c->scale.p, c->z.p);
            int j = 0, batch = 0, pending = -1;
            bool ended = false;
            while (!ended) {
                for (int q = 0; q < kBatch; ++q, ++j) {
                    double* u = V + size_t(j) * size_t(n);
                    const bool last = (j == m) || (j >= 1 && it0 + j >= kc->max_iters);
                    const long q0 = prof_mark(c);
                    if (!last)
                        TRY(matvec_dev(c, c->z.p, c->w.p, nullptr, true, c->scale.p, ad.ctl));
                    const long q1 = prof_mark(c);
                    if (n <= kDots2dMax)
                        launch_dcgs_dots2d(V, n, j, u, last ? nullptr : c->w.p, n, c->partial.p, st, ad.ctl);
                    else
                        launch_dcgs_dots(V, n, j, u, last ? nullptr : c->w.p, n, c->partial.p, st, ad.ctl);
                    launch_reduce_partials(c->partial.p, last ? j + 1 : 2 * j + 3, c->red.p, 0, st, ad.ctl,
                                           dcgs_dots_parts(n));
                    const long q2 = prof_mark(c);
                    launch_arnoldi_step(ad, j, last ? 1 : 0, c->red.p, d_norm, d_coef, bnorm, kc->tolerance, st);
                    const long q3 = prof_mark(c);
                    prof_pair(c, kPhGmMatvec, q0, q1);
                    prof_pair(c, kPhGmDots, q1, q2);
                    prof_pair(c, kPhGmArnoldi, q2, q3);
                    if (last) {
                        ended = true;
                        break;
                    }
                    double* upart = c->partial.p + size_t(2 * m + 8) * kRedBlocks;
                    launch_dcgs_update2(V, n, j, d_coef, u, c->w.p, n, upart, st, ad.ctl);
                    launch_normalize_partials(c->w.p, upart, dcgs_update_parts(n), d_norm,
                                              V + size_t(j + 1) * size_t(n), c->scale.p, c->z.p, n, st, ad.ctl);
                    prof_pair(c, kPhGmUpdate, q3, prof_mark(c));
                }
                TRY(check_launch(c));
                if (ended)
                    break;
                const int slot = batch & 1;
                CK(c, cudaMemcpyAsync(c->h_ctl + 4 * slot, ad.ctl, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
                CK(c, cudaEventRecord(c->ctl_ev[slot], st));
                if (pending >= 0) {
                    CK(c, cudaEventSynchronize(c->ctl_ev[pending]));
                    if (c->h_ctl[4 * pending] != 0)
                        ended = true;
                }
                pending = slot;
                ++batch;
            }
            CK(c, cudaMemcpyAsync(c->h_ctl + 8, ad.ctl, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
            CK(c, cudaStreamSynchronize(st));
            res->iterations = c->h_ctl[9];
            ncols = c->h_ctl[10];
            res->reorthogonalizations = c->h_ctl[11];
            if (ncols > 0) {
                CK(c, cudaMemcpy(R.data(), ad.R, sizeof(double) * size_t(m + 2) * size_t(ncols),
                                 cudaMemcpyDeviceToHost));
                CK(c, cudaMemcpy(gv.data(), ad.gv, sizeof(double) * size_t(ncols + 1), cudaMemcpyDeviceToHost));
            }
        } else {
            bool stop = false;
            for (int j = 0; !stop; ++j) {
                double* u = V + size_t(j) * size_t(n);
                // last step of the cycle: only finalise column j-1
                const bool last = (j == m) || (res->iterations + (j >= 1 ? 1 : 0) >= kc->max_iters);
                if (!last)
                    TRY(apply_op(c->z.p, c->w.p, c->scale.p));  // w = S A S u_j
                launch_dcgs_dots(V, n, j, u, last ? nullptr : c->w.p, n, c->partial.p, st);
                const int rows = last ? j + 1 : 2 * j + 3;
                launch_reduce_partials(c->partial.p, rows, c->red.p, 0, st);
                TRY(check_launch(c));
                CK(c, cudaMemcpyAsync(c->h_red, c->red.p, sizeof(double) * size_t(rows),
                                      cudaMemcpyDeviceToHost, st));
                if (j >= 1)
                    CK(c, cudaMemcpyAsync(c->h_red + o_norm, d_norm, sizeof(double), cudaMemcpyDeviceToHost, st));
                CK(c, cudaStreamSynchronize(st));
                const double* a = c->h_red;
                const double uu = last ? c->h_red[j] : c->h_red[2 * j];
                double aa = 0.0;
                for (int i = 0; i < j; ++i) {
                    av[size_t(i)] = a[i];
                    aa += a[i] * a[i];
                }
                const double rho2 = uu - aa;
                const double rho = rho2 > 0.0 ? std::sqrt(rho2) : 0.0;
                if (j >= 1) {
                    // finalise column j-1: H[j, j-1] held |w'_{j-1}| (the norm u_j was built with)
                    HH(j, j - 1) = c->h_red[o_norm];
                    const double hjj1 = HH(j, j - 1);
                    for (int i = 0; i < j; ++i)
                        HH(i, j - 1) += hjj1 * av[size_t(i)];
                    HH(j, j - 1) = hjj1 * rho;
                    // Givens (linalg.cpp:237-258) on the final column
                    const int k = j - 1;
                    for (int i = 0; i <= j; ++i)
                        RR(i, k) = HH(i, k);
                    for (int i = 0; i < k; ++i) {
                        const double t = cs[size_t(i)] * RR(i, k) + sn[size_t(i)] * RR(i + 1, k);
                        RR(i + 1, k) = -sn[size_t(i)] * RR(i, k) + cs[size_t(i)] * RR(i + 1, k);
                        RR(i, k) = t;
                    }
                    const double den = std::hypot(RR(k, k), RR(k + 1, k));
                    cs[size_t(k)] = den == 0.0 ? 1.0 : RR(k, k) / den;
                    sn[size_t(k)] = den == 0.0 ? 0.0 : RR(k + 1, k) / den;
                    RR(k, k) = den;
                    RR(k + 1, k) = 0.0;
                    gv[size_t(k) + 1] = -sn[size_t(k)] * gv[size_t(k)];
                    gv[size_t(k)] = cs[size_t(k)] * gv[size_t(k)];
                    res->iterations += 1;
                    res->reorthogonalizations += 1;
                    ncols = j;
                    const double est = std::fabs(gv[size_t(k) + 1]);
                    push_hist(est / bnorm);
                    if (est / bnorm <= kc->tolerance || HH(j, j - 1) == 0.0)
                        stop = true;
                }
                if (last || stop)
                    break;
                // tentative column j and the update pass
                const double* b = c->h_red + j;
                const double uw = c->h_red[2 * j + 1];
                double ab = 0.0;
                for (int i = 0; i < j; ++i)
                    ab += av[size_t(i)] * b[i];
                if (!(rho > 0.0)) {
                    stop = true;  // u_j in span(Q): breakdown
                    break;
                }
                const double cj = (uw - ab) / rho;
                for (int i = 0; i <= j; ++i) {
                    double ha = 0.0;
                    for (int l = 0; l < j; ++l)
                        ha += HH(i, l) * av[size_t(l)];
                    HH(i, j) = ((i < j ? b[i] : cj) - ha) / rho;
                }
                const double cr = cj / rho;
                for (int i = 0; i < j; ++i) {
                    h_coef[i] = av[size_t(i)];
                    h_coef[j + i] = b[i] - cr * av[size_t(i)];
                }
                h_coef[2 * j] = 1.0 / rho;
                h_coef[2 * j + 1] = cr;
                CK(c, cudaMemcpyAsync(d_coef, h_coef, sizeof(double) * size_t(2 * j + 2),
                                      cudaMemcpyHostToDevice, st));
                double* upart = c->partial.p + size_t(2 * m + 8) * kRedBlocks;
                if (j == 0)
                    gv[0] *= rho;  // V_0 renormalised by its computed norm in the update pass
                launch_dcgs_update(V, n, j, d_coef, u, c->w.p, n, upart, st);
                launch_reduce_partials(upart, 1, d_norm, 1, st);
                // tentative u_{j+1} = w'/|w'| and z = S u_{j+1}
                launch_normalize(c->w.p, d_norm, V + size_t(j + 1) * size_t(n), n, st, c->scale.p, c->z.p);
                TRY(check_launch(c));
            }
        }
        int j = ncols;
        while (j > 0 && RR(j - 1, j - 1) == 0.0)
            --j;
        for (int i = j - 1; i >= 0; --i) {
            double sacc = gv[size_t(i)];
            for (int k = i + 1; k < j; ++k)
                sacc -= RR(i, k) * yv[size_t(k)];
            yv[size_t(i)] = sacc / RR(i, i);
        }
        if (j > 0) {
            std::copy(yv.begin(), yv.begin() + j, c->h_red);
            CK(c, cudaMemcpyAsync(c->red.p, c->h_red, sizeof(double) * size_t(j),
                                  cudaMemcpyHostToDevice, st));
            launch_basis_combine(V, n, j, c->red.p, c->scale.p, d_x, n, st);
        }
        // recomputed scaled residual r = S (rhs - L x)
        TRY(apply_op(d_x, c->w.p, nullptr));
        launch_scaled_diff(c->scale.p, d_rhs, c->w.p, c->tmp.p, n, st);
        rsrc = c->tmp.p;
        TRY(dot_dev(c, c->tmp.p, c->tmp.p, n, &rnorm, true));
        res->relative_residual = rnorm / bnorm;
        if (res->relative_residual <= kc->tolerance) {
            res->status = 0;
            return pull_hist();
        }
        if (rnorm >= cycle_start) {
            res->status = 2;
            return pull_hist();
        }
    }
    res->status = 1;
    return pull_hist();
}

// ---------------------------------------------------------------- C ABI

extern "C" {

const char* hbgpu_create_error(void) { return g_create_error.c_str(); }

hbgpu_ctx* hbgpu_create(const hbgpu_mesh_desc* d, int* status) {
    auto set = [&](int s, const std::string& m) {
        if (status)
            *status = s;
        g_create_error = m;
    };
    if (!d || d->num_nodes <= 0 || d->num_elements < 0 || !d->conn || !d->dirichlet ||
        (!d->geometry && !d->xyz)) {
        set(HBGPU_ERR_INVALID, "invalid mesh descriptor");
        return nullptr;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set(HBGPU_ERR_CUDA, "no CUDA device: the HB-GLS GPU path has no CPU fallback");
        return nullptr;
    }
    int dev = 0, major = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major < 10) {
        set(HBGPU_ERR_CUDA, "libhbgpu is built for sm_100a (B200); device is older");
        return nullptr;
    }
    auto* c = new hbgpu_ctx;
    c->tool = Tooling::from_env();
    c->nn = d->num_nodes;
    c->ne = d->num_elements;
    c->conn_h.assign(d->conn, d->conn + 4 * size_t(c->ne));
    c->dir_h.assign(d->dirichlet, d->dirichlet + size_t(c->nn));
    for (int k = 0; k < 4 * c->ne; ++k)
        if (d->conn[k] < 0 || d->conn[k] >= c->nn) {
            set(HBGPU_ERR_PARSE, "element references a node out of range");
            delete c;
            return nullptr;
        }
    size_t off = 0;
    for (int p = 0; p < d->num_patches; ++p) {
        HostPatch hp;
        hp.kind = d->patch_kind[p];
        const int nf = d->patch_num_facets[p];
        hp.facets.assign(d->facets + 3 * off, d->facets + 3 * (off + size_t(nf)));
        hp.normals.assign(d->normals + 3 * off, d->normals + 3 * (off + size_t(nf)));
        hp.areas.assign(d->areas + off, d->areas + off + size_t(nf));
        for (double a : hp.areas)
            hp.area += a;
        c->patches.push_back(std::move(hp));
        off += size_t(nf);
    }
    // characteristic length (mesh.cpp:213-224), from signed volumes
    if (c->ne > 0) {
        double total = 0.0;
        if (d->xyz) {
            for (int e = 0; e < c->ne; ++e) {
                const double* x[4];
                for (int a = 0; a < 4; ++a)
                    x[a] = d->xyz + 3 * size_t(d->conn[4 * e + a]);
                const double b0[3] = {x[1][0] - x[0][0], x[1][1] - x[0][1], x[1][2] - x[0][2]};
                const double b1[3] = {x[2][0] - x[0][0], x[2][1] - x[0][1], x[2][2] - x[0][2]};
                const double b2[3] = {x[3][0] - x[0][0], x[3][1] - x[0][1], x[3][2] - x[0][2]};
                const double cr[3] = {b1[1] * b2[2] - b1[2] * b2[1], b1[2] * b2[0] - b1[0] * b2[2],
                                      b1[0] * b2[1] - b1[1] * b2[0]};
                total += (b0[0] * cr[0] + b0[1] * cr[1] + b0[2] * cr[2]) / 6.0;
            }
        } else {
            for (int e = 0; e < c->ne; ++e)
                total += d->geometry[22 * size_t(e) + 12];
        }
        c->h_c = std::cbrt(6.0 * std::sqrt(2.0) * (total / double(c->ne)));
    }
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        set(HBGPU_ERR_CUDA, "cudaStreamCreate failed");
        delete c;
        return nullptr;
    }
    const int st = upload_all(c, d);
    if (st != HBGPU_OK) {
        set(st, c->err);
        hbgpu_destroy(c);
        return nullptr;
    }
    if (status)
        *status = HBGPU_OK;
    return c;
}

void hbgpu_destroy(hbgpu_ctx* c) {
    if (!c)
        return;
    if (c->stream)
        cudaStreamSynchronize(c->stream);
    if (c->h_red)
        cudaFreeHost(c->h_red);
    if (c->h_int)
        cudaFreeHost(c->h_int);
    if (c->h_ctl)
        cudaFreeHost(c->h_ctl);
    for (cudaEvent_t e : c->ctl_ev)
        if (e)
            cudaEventDestroy(e);
    c->arn.release();
    c->arn_ctl.release();
    c->mv_rows.release();
    c->res_ptr.release();
    c->res_node.release();
    c->res_b.release();
    c->res_R.release();
    for (DBuf<double>* b : {&c->geom, &c->H, &c->g, &c->hN, &c->fnormal, &c->farea, &c->state,
                            &c->r, &c->hu, &c->pvals, &c->mass, &c->mass_c, &c->inv, &c->y, &c->out,
                            &c->x, &c->w, &c->z, &c->scale, &c->b, &c->tmp, &c->V, &c->partial, &c->red, &c->rpartial})
        b->release();
    for (DBuf<int>* b : {&c->row_ptr, &c->col_idx, &c->mv_perm, &c->diag_blk, &c->inc_ptr, &c->rpack_ptr, &c->npart_ptr, &c->npart,
                         &c->bnode, &c->bptr, &c->binc, &c->fac, &c->fbc, &c->flag,
                         &c->ideg})
        b->release();
    c->conn.release();
    c->dir.release();
    c->inc_rec.release();
    c->contrib_ptr.release();
    c->contrib.release();
    for (auto& b : c->tb) {
        b.desc.release();
        b.pack.release();
        b.pack_ptr.release();
    }
    c->blkc.release();
    c->blk_order.release();
    c->tgeom.release();
    c->rpack.release();
    for (cudaEvent_t e : c->ev_pool)
        cudaEventDestroy(e);
    if (c->ev_fork)
        cudaEventDestroy(c->ev_fork);
    if (c->ev_join)
        cudaEventDestroy(c->ev_join);
    if (c->stream2)
        cudaStreamDestroy(c->stream2);
    if (c->stream)
        cudaStreamDestroy(c->stream);
    delete c;
}

const char* hbgpu_last_error(const hbgpu_ctx* c) { return c ? c->err.c_str() : ""; }

void* hbgpu_stream(hbgpu_ctx* c) { return c->stream; }

int hbgpu_synchronize(hbgpu_ctx* c) {
    CK(c, cudaStreamSynchronize(c->stream));
    return check_flag(c);
}

int hbgpu_set_basis(hbgpu_ctx* c, int modes, double period) {
    if (modes < 1)
        return fail(c, HBGPU_ERR_PARSE, "spectral basis requires at least one mode (M >= 1)");
    if (!(period > 0.0))
        return fail(c, HBGPU_ERR_PARSE, "spectral basis requires a positive period");
    if (modes > HBGPU_MAX_MODES)
        return fail(c, HBGPU_ERR_INVALID,
                    "spectral basis: M = " + std::to_string(modes) + " exceeds the supported maximum " +
                        std::to_string(HBGPU_MAX_MODES) + " (N = 2M-1 <= " +
                        std::to_string(2 * HBGPU_MAX_MODES - 1) +
                        " time samples; the dense H lives in shared memory)");
    if ((unsigned long long)c->nn * 4ull * (unsigned long long)(2 * modes - 1) >= (1ull << 32))
        return fail(c, HBGPU_ERR_INVALID, "state vector exceeds 2^32 doubles (32-bit element offsets in the gathers)");
    c->M = modes;
    c->N = 2 * modes - 1;
    c->period = period;
    c->omega = 2.0 * M_PI / period;
    const int N = c->N;
    // H = E^-1 Omega E, E(j,k) = e^{-2 pi i j k/N}/N, Omega_kk = i omega m(k) (spectral.cpp:236-256)
    std::vector<double> H(size_t(N) * size_t(N));
    for (int j = 0; j < N; ++j)
        for (int k = 0; k < N; ++k) {
            std::complex<double> acc(0.0, 0.0);
            for (int l = 0; l < N; ++l) {
                const double ph1 = 2.0 * M_PI * double(j) * double(l) / double(N);
                const double ph2 = -2.0 * M_PI * double(l) * double(k) / double(N);
                const std::complex<double> einv(std::cos(ph1), std::sin(ph1));
                const std::complex<double> e(std::cos(ph2) / N, std::sin(ph2) / N);
                const int mm = l < modes ? l : l - N;
                const std::complex<double> om(0.0, c->omega * double(mm));
                acc += einv * om * e;
            }
            H[size_t(j) * size_t(N) + size_t(k)] = acc.real();
        }
    CK(c, c->H.alloc(H.size()));
    CK(c, cudaMemcpyAsync(c->H.p, H.data(), sizeof(double) * H.size(), cudaMemcpyHostToDevice,
                          c->stream));
    const size_t n = size_t(c->state_len());
    for (DBuf<double>* b : {&c->state, &c->r, &c->inv, &c->y, &c->out, &c->x, &c->w, &c->z,
                            &c->scale, &c->b, &c->tmp})
        CK(c, b->alloc(n));
    CK(c, c->hu.alloc(size_t(c->nn) * 3 * size_t(N)));
    c->res_tile = residual_tile(N);
    if (c->tool.res_tile == 1 || c->tool.res_tile == 2 || c->tool.res_tile == 4)
        c->res_tile = c->tool.res_tile;
    CK(c, c->rpartial.alloc(size_t(c->npairs) * 7 * size_t((N + c->res_tile - 1) / c->res_tile) * c->res_tile));
    {
        const size_t rs = residual_smem_bytes(c->max_nloc, c->max_rpack, c->res_tile);
        CK(c, configure_residual_smem(rs, c->res_tile));
        int per_sm = 0, nsm = 0, dev = 0;
        CK(c, cudaGetDevice(&dev));
        CK(c, cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        CK(c, residual_occupancy(&per_sm, rs, c->res_tile));
        c->res_grid = nsm * std::max(1, per_sm);
    }
    CK(c, c->pvals.alloc(size_t(c->nnz) * 8 * size_t(N)));
    CK(c, c->mass.alloc(size_t(c->nnz)));
    CK(c, c->mass_c.alloc(size_t(c->nnz)));
    CK(c, c->g.alloc(size_t(c->nn) * 3 * size_t(N)));
    CK(c, cudaMemsetAsync(c->g.p, 0, sizeof(double) * size_t(c->nn) * 3 * size_t(N), c->stream));
    c->g_h.assign(size_t(c->nn) * 3 * size_t(N), 0.0);
    c->V.release();
    c->p_valid = c->inv_valid = false;
    c->mass_valid = false;
    {
        // per bucket: the persistent row pipeline.  CTA width w (32 ... 512) is
        // picked by a throughput score: useful thread fraction of the row's
        // phase-1 items (incidences x samples) times min(1, resident warps / 12),
        // residency limited by shared memory (whole time series per CTA), 128
        // registers per thread and 32 CTAs per SM; ties go to the narrower CTA.
        // If no width holds the whole series, 512 threads and the largest tile
        // that fits.  Rows whose neighbour records cannot be buffered at all use
        // the tiled row kernel.
        size_t mx = 0, mxp[5] = {0, 0, 0, 0, 0};
        int dev = 0, nsm = 0;
        // test knob: HBGPU_TANGENT_KERNEL=rows forces the row-kernel fallback
        const bool force_rows = c->tool.tangent_rows;
        CK(c, cudaGetDevice(&dev));
        CK(c, cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const int widths[5] = {32, 64, 128, 256, 512};
        for (auto& b : c->tb) {
            if (!b.count)
                continue;
            auto ps = [&](int nt) { return tangent_pipe_smem(b.max_pack, b.max_inc, b.max_blk, N, nt); };
            b.pipe = false;
            if (TAN_PIPE && !force_rows) {
                const double items = double(b.max_inc) * N;
                double best = 0.0;
                for (int w : widths) {
                    const size_t sm = ps(N);
                    if (sm > size_t(227 * 1024))
                        continue;
                    const int by_smem = int(size_t(228 * 1024) / (sm + 1024));
                    const int by_regs = 65536 / (w * 128);
                    const int ctas = std::min({32, by_smem, by_regs});
                    if (ctas < 1)
                        continue;
                    const double rounds = std::ceil(items / w);
                    const double score = items / (rounds * w) * std::min(1.0, ctas * (w / 32) / 12.0);
                    if (score > best * 1.0001) {
                        best = score;
                        b.pipe = true;
                        b.threads = w;
                        b.nt = N;
                    }
                }
                // tooling: HBGPU_TAN_WIDTH forces the CTA width of every pipe bucket
                if (c->tool.tan_width) {
                    const int w = c->tool.tan_width;
                    if (b.pipe && std::find(widths, widths + 5, w) != widths + 5 && ps(b.nt) <= size_t(227 * 1024))
                        b.threads = w;
                }
                if (!b.pipe) {
                    int nt = N;
                    while (nt > 1 && ps(nt) > size_t(226 * 1024))
                        nt = (nt + 1) / 2;
                    if (ps(nt) <= size_t(226 * 1024)) {
                        b.pipe = true;
                        b.threads = 512;
                        b.nt = nt;
                    }
                }
            }
            if (b.pipe) {
                b.smem = ps(b.nt);
                const int w = int(std::find(widths, widths + 5, b.threads) - widths);
                mxp[w] = std::max(mxp[w], b.smem);
                continue;
            }
            int nt = N;
            const int dp = (b.max_inc + kTanPart - 1) / kTanPart;
            while (nt > 1 && tangent_row_smem(b.max_inc, b.max_blk, dp, nt) > TAN_SMEM_KB * 1024)
                nt = (nt + 1) / 2;
            b.smem = tangent_row_smem(b.max_inc, b.max_blk, dp, nt);
            b.nt = nt;
            mx = std::max(mx, b.smem);
        }
        if (mx > 227 * 1024)
            return fail(c, HBGPU_ERR_INVALID, "node valence too high for the tangent row kernel");
        if (mx)
            CK(c, configure_tangent_row_smem(mx));
        for (int w = 0; w < 5; ++w)
            if (mxp[w])
                CK(c, configure_tangent_pipe_smem(widths[w], mxp[w]));
        for (auto& b : c->tb) {
            if (!b.count || !b.pipe)
                continue;
            int per_sm = 0;
            CK(c, tangent_pipe_occupancy(b.threads, &per_sm, b.smem));
            if (per_sm < 1)
                return fail(c, HBGPU_ERR_INVALID, "tangent pipeline does not fit on an SM");
            const int tiles = (N + b.nt - 1) / b.nt;
            b.grid = std::max(1, std::min(b.count, (nsm * per_sm + tiles - 1) / tiles));
        }
    }
    // clear previous Neumann data sized for another N
    c->hN.release();
    c->h_h.clear();
    c->bc_patch.clear();
    c->nbnodes = 0;
    CK(c, cudaStreamSynchronize(c->stream));
    return HBGPU_OK;
}

int hbgpu_set_fluid(hbgpu_ctx* c, double rho, double mu) {
    if (!(rho > 0.0) || !(mu > 0.0))
        return fail(c, HBGPU_ERR_PARSE, "fluid density and viscosity must be strictly positive");
    c->rho = rho;
    c->mu = mu;
    c->mass_valid = false;
    return HBGPU_OK;
}

int hbgpu_set_assembly_config(hbgpu_ctx* c, int tau_mode, double pseudo_dt, double pseudo_c1,
                              int backflow_in_tangent) {
    c->tau_mode = tau_mode == 1 ? 1 : 0;
    c->pseudo_dt = (pseudo_dt > 0.0 && std::isfinite(pseudo_dt))
                       ? pseudo_dt
                       : std::numeric_limits<double>::infinity();
    c->pseudo_c1 = pseudo_c1;
    c->backflow_tangent = backflow_in_tangent;
    return HBGPU_OK;
}

int hbgpu_set_bcs(hbgpu_ctx* c, const double* dirichlet_g, int n_neumann, const int* neumann_patch,
                  const double* neumann_h, double backflow_beta) {
    TRY(ensure_basis(c));
    // validate everything before any context state changes
    if (n_neumann < 0 || (n_neumann > 0 && (!neumann_patch || !neumann_h)))
        return fail(c, HBGPU_ERR_INVALID, "set_bcs: bad Neumann arguments");
    for (int k = 0; k < n_neumann; ++k)
        if (neumann_patch[k] < 0 || neumann_patch[k] >= int(c->patches.size()))
            return fail(c, HBGPU_ERR_INVALID, "Neumann entry references an unknown patch");
    const int N = c->N;
    const size_t gl = size_t(c->nn) * 3 * size_t(N);
    if (dirichlet_g)
        c->g_h.assign(dirichlet_g, dirichlet_g + gl);
    else
        c->g_h.assign(gl, 0.0);
    CK(c, cudaMemcpyAsync(c->g.p, c->g_h.data(), sizeof(double) * gl, cudaMemcpyHostToDevice,
                          c->stream));
    c->beta = backflow_beta;
    c->bc_patch.assign(neumann_patch, neumann_patch + n_neumann);
    c->h_h.assign(neumann_h, neumann_h + size_t(n_neumann) * size_t(N));
    // facet arrays over the Neumann list (assembly.cpp:537-539 order) and
    // per-node incidence lists in that order
    std::vector<int> fac, fbc;
    std::vector<double> fnorm, farea;
    for (int k = 0; k < n_neumann; ++k) {
        const HostPatch& p = c->patches[size_t(neumann_patch[k])];
        for (size_t f = 0; f < p.areas.size(); ++f) {
            for (int v = 0; v < 3; ++v) {
                fac.push_back(p.facets[3 * f + size_t(v)]);
                fnorm.push_back(p.normals[3 * f + size_t(v)]);
            }
            farea.push_back(p.areas[f]);
            fbc.push_back(k);
        }
    }
    const int nf = int(farea.size());
    std::vector<int> cnt(size_t(c->nn) + 1, 0);
    for (int f = 0; f < nf; ++f)
        for (int v = 0; v < 3; ++v)
            cnt[size_t(fac[3 * size_t(f) + size_t(v)]) + 1] += 1;
    std::vector<int> bnode, bptr{0}, binc;
    std::vector<int> start(size_t(c->nn), -1);
    for (int A = 0; A < c->nn; ++A)
        if (cnt[size_t(A) + 1] > 0) {
            start[size_t(A)] = bptr.back();
            bnode.push_back(A);
            bptr.push_back(bptr.back() + cnt[size_t(A) + 1]);
        }
    binc.assign(size_t(bptr.back()), 0);
    std::vector<int> fillp(start);
    for (int f = 0; f < nf; ++f)
        for (int v = 0; v < 3; ++v) {
            const int A = fac[3 * size_t(f) + size_t(v)];
            binc[size_t(fillp[size_t(A)]++)] = f * 4 + v;
        }
    c->nbnodes = int(bnode.size());
    if (nf > 0) {
        CK(c, c->fac.alloc(fac.size()));
        CK(c, c->fbc.alloc(fbc.size()));
        CK(c, c->fnormal.alloc(fnorm.size()));
        CK(c, c->farea.alloc(farea.size()));
        CK(c, c->bnode.alloc(bnode.size()));
        CK(c, c->bptr.alloc(bptr.size()));
        CK(c, c->binc.alloc(binc.size()));
        CK(c, c->hN.alloc(c->h_h.size()));
        cudaStream_t st = c->stream;
        CK(c, cudaMemcpyAsync(c->fac.p, fac.data(), sizeof(int) * fac.size(), cudaMemcpyHostToDevice, st));
        CK(c, cudaMemcpyAsync(c->fbc.p, fbc.data(), sizeof(int) * fbc.size(), cudaMemcpyHostToDevice, st));
        CK(c, cudaMemcpyAsync(c->fnormal.p, fnorm.data(), sizeof(double) * fnorm.size(), cudaMemcpyHostToDevice, st));
        CK(c, cudaMemcpyAsync(c->farea.p, farea.data(), sizeof(double) * farea.size(), cudaMemcpyHostToDevice, st));
        CK(c, cudaMemcpyAsync(c->bnode.p, bnode.data(), sizeof(int) * bnode.size(), cudaMemcpyHostToDevice, st));
        CK(c, cudaMemcpyAsync(c->bptr.p, bptr.data(), sizeof(int) * bptr.size(), cudaMemcpyHostToDevice, st));
        CK(c, cudaMemcpyAsync(c->binc.p, binc.data(), sizeof(int) * binc.size(), cudaMemcpyHostToDevice, st));
        CK(c, cudaMemcpyAsync(c->hN.p, c->h_h.data(), sizeof(double) * c->h_h.size(), cudaMemcpyHostToDevice, st));
    }
    CK(c, cudaStreamSynchronize(c->stream));
    return HBGPU_OK;
}

int hbgpu_set_resistance(hbgpu_ctx* c, int n, const int* patch, const double* R) {
    if (n < 0 || (n > 0 && (!patch || !R)))
        return fail(c, HBGPU_ERR_INVALID, "set_resistance: bad arguments");
    std::vector<int> ptr{0}, node;
    std::vector<double> b, rv;
    for (int k = 0; k < n; ++k) {
        if (patch[k] < 0 || patch[k] >= int(c->patches.size()) || c->patches[size_t(patch[k])].kind != 1)
            return fail(c, HBGPU_ERR_INVALID, "set_resistance: patch " + std::to_string(patch[k]) +
                                                  " is not a Neumann patch");
        if (R[k] == 0.0)
            continue;
        const HostPatch& p = c->patches[size_t(patch[k])];
        // b_A = sum over A's facets (facet order) of area/3 * normal
        std::vector<int> local(static_cast<size_t>(c->nn), -1);
        const size_t base = node.size();
        for (size_t f = 0; f < p.areas.size(); ++f)
            for (int a = 0; a < 3; ++a) {
                const int A = p.facets[3 * f + size_t(a)];
                if (local[size_t(A)] < 0) {
                    local[size_t(A)] = int(node.size() - base);
                    node.push_back(A);
                    b.insert(b.end(), {0.0, 0.0, 0.0});
                }
                double* bk = b.data() + 3 * (base + size_t(local[size_t(A)]));
                for (int i = 0; i < 3; ++i)
                    bk[i] += p.areas[f] / 3.0 * p.normals[3 * f + size_t(i)];
            }
        ptr.push_back(int(node.size()));
        rv.push_back(R[k]);
    }
    c->nres = int(rv.size());
    if (c->nres > 0) {
        CK(c, c->res_ptr.alloc(ptr.size()));
        CK(c, c->res_node.alloc(node.size()));
        CK(c, c->res_b.alloc(b.size()));
        CK(c, c->res_R.alloc(rv.size()));
        CK(c, cudaMemcpy(c->res_ptr.p, ptr.data(), sizeof(int) * ptr.size(), cudaMemcpyHostToDevice));
        CK(c, cudaMemcpy(c->res_node.p, node.data(), sizeof(int) * node.size(), cudaMemcpyHostToDevice));
        CK(c, cudaMemcpy(c->res_b.p, b.data(), sizeof(double) * b.size(), cudaMemcpyHostToDevice));
        CK(c, cudaMemcpy(c->res_R.p, rv.data(), sizeof(double) * rv.size(), cudaMemcpyHostToDevice));
    }
    return HBGPU_OK;
}

int hbgpu_sizes(const hbgpu_ctx* c, int* nn, int* ne, int* N, long long* nnz, long long* slen) {
    if (nn) *nn = c->nn;
    if (ne) *ne = c->ne;
    if (N) *N = c->N;
    if (nnz) *nnz = c->nnz;
    if (slen) *slen = c->state_len();
    return HBGPU_OK;
}

int hbgpu_get_pattern(hbgpu_ctx* c, int* row_ptr, int* col_idx) {
    if (row_ptr)
        CK(c, cudaMemcpy(row_ptr, c->row_ptr.p, sizeof(int) * (size_t(c->nn) + 1), cudaMemcpyDeviceToHost));
    if (col_idx)
        CK(c, cudaMemcpy(col_idx, c->col_idx.p, sizeof(int) * size_t(c->nnz), cudaMemcpyDeviceToHost));
    return HBGPU_OK;
}

int hbgpu_get_geometry(hbgpu_ctx* c, double* geometry) {
    CK(c, cudaMemcpy(geometry, c->geom.p, sizeof(double) * 22 * size_t(c->ne), cudaMemcpyDeviceToHost));
    return HBGPU_OK;
}

int hbgpu_assemble_residual_dev(hbgpu_ctx* c, const double* d_state, double* d_r) {
    TRY(ensure_basis(c));
    return residual_dev(c, d_state, d_r);
}

int hbgpu_assemble_residual(hbgpu_ctx* c, const double* state, double* residual) {
    TRY(ensure_basis(c));
    const size_t n = size_t(c->state_len());
    CK(c, cudaMemcpyAsync(c->state.p, state, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    TRY(residual_dev(c, c->state.p, c->r.p));
    CK(c, cudaMemcpyAsync(residual, c->r.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return check_flag(c);
}

// Residual and tangent of the same state, the tangent on the second stream so
// the two latency-bound kernels share the SMs; ordered on ctx->stream after.
// With host_r the residual's copy to the host is queued right behind the
// residual, so it overlaps the tangent.
// Fused assembly: the residual pass also writes the tangent's element
// summaries; the tangent rows then run without recomputing them.
static int assemble_both(hbgpu_ctx* c, const double* d_state, double* d_r, double* host_r = nullptr) {
    if (host_r) {
        // host copy-back wanted: residual first, then the tangent on the second
        // stream while the residual travels back (concurrent kernels would finish
        // together and leave the copy exposed)
        TRY(residual_dev(c, d_state, d_r));
        CK(c, cudaEventRecord(c->ev_fork, c->stream));
        CK(c, cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
        CK(c, cudaMemcpyAsync(host_r, d_r, sizeof(double) * size_t(c->state_len()), cudaMemcpyDeviceToHost,
                              c->stream));
        cudaStream_t main = c->stream;
        c->stream = c->stream2;
        const int st = tangent_dev(c, d_state);
        c->stream = main;
        TRY(st);
        CK(c, cudaEventRecord(c->ev_join, c->stream2));
        CK(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
        return HBGPU_OK;
    }
    // residual and tangent concurrently on the context's two streams
    CK(c, cudaEventRecord(c->ev_fork, c->stream));
    CK(c, cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
    cudaStream_t main = c->stream;
    c->stream = c->stream2;
    const int st = tangent_dev(c, d_state);
    c->stream = main;
    TRY(st);
    TRY(residual_dev(c, d_state, d_r));
    CK(c, cudaEventRecord(c->ev_join, c->stream2));
    CK(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    return HBGPU_OK;
}

int hbgpu_assemble(hbgpu_ctx* c, const double* state, double* residual) {
    TRY(ensure_basis(c));
    const size_t n = size_t(c->state_len());
    CK(c, cudaMemcpyAsync(c->state.p, state, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    TRY(assemble_both(c, c->state.p, c->r.p, residual));
    CK(c, cudaStreamSynchronize(c->stream));
    return check_flag(c);
}

int hbgpu_assemble_dev(hbgpu_ctx* c, const double* d_state, double* d_residual) {
    TRY(ensure_basis(c));
    return assemble_both(c, d_state, d_residual);
}

int hbgpu_assemble_tangent_dev(hbgpu_ctx* c, const double* d_state) {
    TRY(ensure_basis(c));
    return tangent_dev(c, d_state);
}

int hbgpu_assemble_tangent(hbgpu_ctx* c, const double* state, double* pvals) {
    TRY(ensure_basis(c));
    const size_t n = size_t(c->state_len());
    CK(c, cudaMemcpyAsync(c->state.p, state, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    TRY(tangent_dev(c, c->state.p));
    if (pvals)
        CK(c, cudaMemcpyAsync(pvals, c->pvals.p, sizeof(double) * size_t(c->nnz) * 8 * size_t(c->N),
                              cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return check_flag(c);
}

int hbgpu_assemble_mass(hbgpu_ctx* c, double* mass) {
    TRY(ensure_basis(c));
    TRY(mass_dev(c));
    if (mass)
        CK(c, cudaMemcpyAsync(mass, c->mass.p, sizeof(double) * size_t(c->nnz), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return HBGPU_OK;
}

int hbgpu_set_mass(hbgpu_ctx* c, const double* mass) {
    TRY(ensure_basis(c));
    CK(c, cudaMemcpyAsync(c->mass.p, mass, sizeof(double) * size_t(c->nnz), cudaMemcpyHostToDevice,
                          c->stream));
    launch_mask_mass(c->mass.p, c->row_ptr.p, c->col_idx.p, c->dir.p, c->nn, c->mass_c.p, c->stream);
    TRY(check_launch(c));
    CK(c, cudaStreamSynchronize(c->stream));
    c->mass_valid = true;
    return HBGPU_OK;
}

int hbgpu_set_pvals(hbgpu_ctx* c, const double* pvals) {
    TRY(ensure_basis(c));
    CK(c, cudaMemcpyAsync(c->pvals.p, pvals, sizeof(double) * size_t(c->nnz) * 8 * size_t(c->N),
                          cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    c->p_valid = true;
    c->inv_valid = false;
    return HBGPU_OK;
}

double* hbgpu_pvals_dev(hbgpu_ctx* c) { return c->pvals.p; }

int hbgpu_get_pvals(hbgpu_ctx* c, double* pvals) {
    if (!c->p_valid)
        return fail(c, HBGPU_ERR_INVALID, "get_pvals before assemble_tangent / set_pvals");
    CK(c, cudaStreamSynchronize(c->stream));
    CK(c, cudaMemcpy(pvals, c->pvals.p, sizeof(double) * size_t(c->nnz) * 8 * size_t(c->N), cudaMemcpyDeviceToHost));
    return HBGPU_OK;
}

int hbgpu_get_pvals_rows(hbgpu_ctx* c, int nrows, const int* rows, double* out) {
    if (!c->p_valid)
        return fail(c, HBGPU_ERR_INVALID, "get_pvals_rows before assemble_tangent / set_pvals");
    if (nrows < 0 || (nrows > 0 && (!rows || !out)))
        return fail(c, HBGPU_ERR_INVALID, "get_pvals_rows: bad arguments");
    CK(c, cudaStreamSynchronize(c->stream));
    const size_t seg = 8 * size_t(c->N);
    size_t off = 0;
    for (int k = 0; k < nrows; ++k) {
        const int A = rows[k];
        if (A < 0 || A >= c->nn)
            return fail(c, HBGPU_ERR_INVALID, "get_pvals_rows: node out of range");
        const size_t r0 = size_t(c->row_ptr_h[size_t(A)]), r1 = size_t(c->row_ptr_h[size_t(A) + 1]);
        CK(c, cudaMemcpyAsync(out + off, c->pvals.p + r0 * seg, sizeof(double) * (r1 - r0) * seg,
                              cudaMemcpyDeviceToHost, c->stream));
        off += (r1 - r0) * seg;
    }
    CK(c, cudaStreamSynchronize(c->stream));
    return HBGPU_OK;
}

int hbgpu_matvec_dev(hbgpu_ctx* c, const double* d_y, double* d_out) {
    TRY(ensure_basis(c));
    return matvec_dev(c, d_y, d_out, nullptr, true);
}

int hbgpu_bsr_matvec_dev(hbgpu_ctx* c, const double* d_y, double* d_out) {
    TRY(ensure_basis(c));
    return matvec_dev(c, d_y, d_out, nullptr, false);
}

static int host_matvec(hbgpu_ctx* c, const double* y, double* out, bool with_c) {
    TRY(ensure_basis(c));
    const size_t n = size_t(c->state_len());
    CK(c, cudaMemcpyAsync(c->y.p, y, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    TRY(matvec_dev(c, c->y.p, c->out.p, nullptr, with_c));
    CK(c, cudaMemcpyAsync(out, c->out.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return HBGPU_OK;
}

int hbgpu_matvec(hbgpu_ctx* c, const double* y, double* out) { return host_matvec(c, y, out, true); }
int hbgpu_bsr_matvec(hbgpu_ctx* c, const double* y, double* out) { return host_matvec(c, y, out, false); }

int hbgpu_jacobi_dev(hbgpu_ctx* c, int* degenerate) {
    TRY(ensure_basis(c));
    return jacobi_dev(c, degenerate);
}

int hbgpu_jacobi(hbgpu_ctx* c, double* inv_diag, int* degenerate) {
    TRY(ensure_basis(c));
    TRY(jacobi_dev(c, degenerate));
    if (inv_diag) {
        CK(c, cudaMemcpyAsync(inv_diag, c->inv.p, sizeof(double) * size_t(c->state_len()),
                              cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
    }
    return HBGPU_OK;
}

int hbgpu_gmres_dev(hbgpu_ctx* c, const double* d_rhs, const hbgpu_krylov_cfg* cfg, double* d_x,
                    hbgpu_krylov_result* result, double* history, int hcap) {
    TRY(ensure_basis(c));
    if (!c->inv_valid)
        TRY(jacobi_dev(c, nullptr));
    const long p0 = prof_mark(c);
    const int st = gmres_dev(c, d_rhs, c->inv.p, cfg, d_x, result, history, hcap);
    prof_pair(c, kPhGmres, p0, prof_mark(c));
    return st;
}

int hbgpu_profile_enable(hbgpu_ctx* c, int on) {
    CK(c, cudaStreamSynchronize(c->stream));
    c->prof = on != 0;
    c->ev_used = 0;
    c->pairs.clear();
    return HBGPU_OK;
}

int hbgpu_profile_read(hbgpu_ctx* c, int nphase, double* ms, int* count) {
    CK(c, cudaStreamSynchronize(c->stream));
    for (int k = 0; k < nphase; ++k) {
        ms[k] = 0.0;
        count[k] = 0;
    }
    for (const auto& p : c->pairs) {
        if (p.phase >= nphase)
            continue;
        float t = 0.0f;
        CK(c, cudaEventElapsedTime(&t, c->ev_pool[p.e0], c->ev_pool[p.e1]));
        ms[p.phase] += double(t);
        count[p.phase] += 1;
    }
    return HBGPU_OK;
}

long long hbgpu_kernel_launches(void) { return g_launches.load(); }

int hbgpu_fp64_peak(double* tflops) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = nsm * 4, threads = 256, iters = 16384;
    double* d = nullptr;
    if (cudaMalloc(&d, sizeof(double)) != cudaSuccess)
        return HBGPU_ERR_CUDA;
    float ms = 0.0f;
    const cudaError_t e = run_fp64_peak(blocks, threads, iters, d, &ms);
    cudaFree(d);
    if (e != cudaSuccess)
        return HBGPU_ERR_CUDA;
    *tflops = 2.0 * 16.0 * double(iters) * blocks * threads / (double(ms) * 1e-3) / 1e12;
    return HBGPU_OK;
}

int hbgpu_gmres_apply(hbgpu_ctx* c, hbgpu_apply_fn apply, void* user, long long n, const double* rhs,
                      const double* inv_diag, const hbgpu_krylov_cfg* cfg, double* x,
                      hbgpu_krylov_result* result, double* history, int hcap) {
    TRY(ensure_basis(c));
    if (!apply || !rhs || !inv_diag || !cfg || !x || !result || n <= 0 || n > c->state_len())
        return fail(c, HBGPU_ERR_INVALID, "gmres_apply: bad arguments (need 0 < n <= the context's state length)");
    c->host_in.resize(size_t(n));
    c->host_out.resize(size_t(n));
    CK(c, cudaMemcpyAsync(c->inv.p, inv_diag, sizeof(double) * size_t(n), cudaMemcpyHostToDevice, c->stream));
    // rhs in its own buffer: gmres_dev overwrites c->b with the scaled rhs and
    // reads the unscaled one again for the true residual of every cycle
    CK(c, cudaMemcpyAsync(c->y.p, rhs, sizeof(double) * size_t(n), cudaMemcpyHostToDevice, c->stream));
    c->host_op = apply;
    c->host_op_user = user;
    c->host_n = long(n);
    const int st = gmres_dev(c, c->y.p, c->inv.p, cfg, c->x.p, result, history, hcap);
    c->host_op = nullptr;
    c->host_op_user = nullptr;
    c->inv_valid = false;  // the context's Jacobi vector was overwritten
    TRY(st);
    CK(c, cudaMemcpy(x, c->x.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost));
    return HBGPU_OK;
}

int hbgpu_gmres(hbgpu_ctx* c, const double* rhs, const double* inv_diag, const hbgpu_krylov_cfg* cfg,
                double* x, hbgpu_krylov_result* result, double* history, int hcap) {
    TRY(ensure_basis(c));
    const size_t n = size_t(c->state_len());
    if (inv_diag) {
        CK(c, cudaMemcpyAsync(c->inv.p, inv_diag, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        c->inv_valid = true;
    } else if (!c->inv_valid) {
        TRY(jacobi_dev(c, nullptr));
    }
    CK(c, cudaMemcpyAsync(c->y.p, rhs, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    TRY(gmres_dev(c, c->y.p, c->inv.p, cfg, c->x.p, result, history, hcap));
    CK(c, cudaMemcpyAsync(x, c->x.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return HBGPU_OK;
}

// solve_harmonic (hb_solver.cpp:113-221)
// The Newton loop of solve_harmonic; every exit (including a failed CUDA call
// or launch) returns through hbgpu_solve_harmonic, which fills the log/info
// and the state as the reference's partial ConvergenceLog would be.
extern "C++" {
template <class LogFn>
static int solve_harmonic_run(hbgpu_ctx* c, const hbgpu_solver_cfg* cfg, hbgpu_solve_info& inf,
                              LogFn&& log) {
    const int N = c->N;
    const long n = long(c->state_len());
    cudaStream_t st = c->stream;
    auto finish = [](int code) { return code; };

    // rest + Dirichlet data + outlet pressure level (hb_solver.cpp:119-132,
    // assembly.cpp:415-441)
    CK(c, cudaMemsetAsync(c->state.p, 0, sizeof(double) * size_t(n), st));
    launch_install_dirichlet(c->g.p, c->dir.p, c->nn, N, c->state.p, st);
    double wsum = 0.0, acc = 0.0;
    for (size_t k = 0; k < c->bc_patch.size(); ++k) {
        double hbar = 0.0;
        for (int m = 0; m < N; ++m)
            hbar += c->h_h[k * size_t(N) + size_t(m)];
        hbar /= double(N);
        const double area = c->patches[size_t(c->bc_patch[k])].area;
        acc += area * (-hbar);
        wsum += area;
    }
    const double p0 = wsum > 0.0 ? acc / wsum : 0.0;
    if (p0 != 0.0)
        launch_fill_pressure(p0, c->nn, N, c->state.p, st);
    TRY(check_launch(c));

    // pseudo-time step (hb_solver.cpp:28-56,86-111)
    double u_c = 0.0;
    bool has_inlet = false;
    for (const HostPatch& p : c->patches) {
        if (p.kind != 0 || !(p.area > 0.0))
            continue;
        has_inlet = true;
        for (int m = 0; m < N; ++m) {
            double q = 0.0;
            for (size_t f = 0; f < p.areas.size(); ++f) {
                const double w = p.areas[f] / 3.0;
                for (int qp = 0; qp < 3; ++qp) {
                    double un = 0.0;
                    for (int a = 0; a < 3; ++a) {
                        const double sa = qp == a ? 2.0 / 3.0 : 1.0 / 6.0;
                        const int A = p.facets[3 * f + size_t(a)];
                        for (int i = 0; i < 3; ++i)
                            un += sa * c->g_h[(size_t(A) * 3 + size_t(i)) * size_t(N) + size_t(m)] *
                                  p.normals[3 * f + size_t(i)];
                    }
                    q += w * un;
                }
            }
            u_c = std::max(u_c, std::fabs(q) / p.area);
        }
    }
    double dt = cfg->pseudo_dt;
    if (!(dt > 0.0))
        dt = u_c <= 0.0 ? c->period / double(N) : c->h_c / u_c;
    if (!has_inlet)
        return finish(fail(c, HBGPU_ERR_GEOMETRY, "CFL number needs a Dirichlet inlet patch with positive area"));
    inf.pseudo_dt = dt;
    inf.cfl = u_c * dt / c->h_c;
    // a fresh AssemblyConfig per solve (hb_solver.cpp:140-146): pseudo_c1 = 1.5
    c->tau_mode = cfg->tau_mode;
    c->pseudo_dt = dt;
    c->pseudo_c1 = 1.5;
    c->backflow_tangent = cfg->backflow_in_tangent;

    {
        Timer t;
        TRY(mass_dev(c));
        CK(c, cudaStreamSynchronize(st));
        inf.assembly_seconds += t.seconds();
    }
    const double target = std::pow(10.0, -cfg->newton_tol_orders);
    double r0 = 0.0;
    std::vector<double> hist;
    for (int iter = 0; iter <= cfg->max_newton_iters; ++iter) {
        Timer t_iter;
        Timer t0;
        // residual and (speculatively) the tangent of this iterate, concurrently;
        // the tangent is unused only on the final iteration
        int s = assemble_both(c, c->state.p, c->r.p);
        if (s != HBGPU_OK)
            return finish(s);
        double res = 0.0;
        s = dot_dev(c, c->r.p, c->r.p, n, &res, true);
        if (s != HBGPU_OK)
            return finish(s);
        s = check_flag(c);
        if (s != HBGPU_OK)
            return finish(s);
        inf.assembly_seconds += t0.seconds();
        if (!std::isfinite(res)) {
            log(iter, res, res / (r0 > 0 ? r0 : 1.0), 0, t_iter.seconds());
            return finish(fail(c, HBGPU_ERR_DIVERGENCE, "residual is not finite at iteration " + std::to_string(iter)));
        }
        if (iter == 0)
            r0 = res;
        const double rel = iter == 0 ? 1.0 : (r0 > 0.0 ? res / r0 : 0.0);
        if (r0 <= 1e-30 || rel <= target) {
            log(iter, res, rel, 0, t_iter.seconds());
            inf.converged = 1;
            break;
        }
        if (rel > cfg->divergence_ratio) {
            log(iter, res, rel, 0, t_iter.seconds());
            return finish(fail(c, HBGPU_ERR_DIVERGENCE, "nonlinear solve diverged: residual ratio " +
                                                             std::to_string(rel) + " at iteration " +
                                                             std::to_string(iter)));
        }
        if (iter == cfg->max_newton_iters) {
            log(iter, res, rel, 0, t_iter.seconds());
            break;
        }
        Timer t2;
        s = jacobi_dev(c, nullptr);
        hbgpu_krylov_result kr{};
        if (s == HBGPU_OK)
            s = gmres_dev(c, c->r.p, c->inv.p, &cfg->krylov, c->x.p, &kr, nullptr, 0);
        if (s != HBGPU_OK)
            return finish(s);
        inf.linear_seconds += t2.seconds();
        if (kr.status == 2)
            return finish(fail(c, HBGPU_ERR_STAGNATION,
                               "GMRES stagnated at Newton iteration " + std::to_string(iter) +
                                   " (relative residual " + std::to_string(kr.relative_residual) + ")"));
        launch_newton_update(c->x.p, c->dir.p, c->nn, N, c->state.p, st);
        TRY(check_launch(c));
        CK(c, cudaStreamSynchronize(st));
        log(iter, res, rel, kr.iterations, t_iter.seconds());
    }
    return finish(HBGPU_OK);
}
}  // extern "C++"

int hbgpu_solve_harmonic(hbgpu_ctx* c, const hbgpu_solver_cfg* cfg, double* state_out,
                         hbgpu_solve_info* info, int cap, int* log_iter, double* log_res,
                         double* log_rel, int* log_lin, double* log_sec) {
    TRY(ensure_basis(c));
    if (!cfg)
        return fail(c, HBGPU_ERR_INVALID, "solve_harmonic: null config");
    Timer total;
    hbgpu_solve_info inf{};
    auto log = [&](int iter, double res, double rel, int lin, double sec) {
        if (!c->tool.solve_progress.empty()) {  // tooling: the ConvergenceLog rows as they are produced
            if (FILE* f = std::fopen(c->tool.solve_progress.c_str(), "a")) {
                std::fprintf(f, "%d,%.17g,%.17g,%d,%.6f\n", iter, res, rel, lin, sec);
                std::fclose(f);
            }
        }
        if (inf.entries < cap) {
            if (log_iter) log_iter[inf.entries] = iter;
            if (log_res) log_res[inf.entries] = res;
            if (log_rel) log_rel[inf.entries] = rel;
            if (log_lin) log_lin[inf.entries] = lin;
            if (log_sec) log_sec[inf.entries] = sec;
            inf.entries += 1;
        }
    };
    // the solve owns its AssemblyConfig; the caller's is restored afterwards
    const int tau0 = c->tau_mode, bf0 = c->backflow_tangent;
    const double dt0 = c->pseudo_dt, c10 = c->pseudo_c1;
    const int code = solve_harmonic_run(c, cfg, inf, log);
    c->tau_mode = tau0;
    c->backflow_tangent = bf0;
    c->pseudo_dt = dt0;
    c->pseudo_c1 = c10;
    inf.total_seconds = total.seconds();
    if (info)
        *info = inf;
    if (state_out) {
        const cudaError_t e = cudaMemcpy(state_out, c->state.p, sizeof(double) * size_t(c->state_len()),
                                         cudaMemcpyDeviceToHost);
        if (e != cudaSuccess && code == HBGPU_OK)
            return fail(c, HBGPU_ERR_CUDA, std::string("solve_harmonic state copy: ") + cudaGetErrorString(e));
    }
    return code;
}


}  // extern "C"

// ---------------------------------------------------------------- time solver
// solve_time (time_solver.cpp:269-485) on the device.  The Newton loop of
// each step follows newton_step (time_solver.cpp:354-455) statement by
// statement; the state lives on the device, the host keeps the scalars
// (residual norms, omega_hat) and calls the Dirichlet callback per step.
namespace {
struct TimeBufs {
    DBuf<double> u, ud, p, nu, nud, np, ual, aal, g, gd, s4, elem, w, prev;
    ~TimeBufs() {
        for (DBuf<double>* b : {&u, &ud, &p, &nu, &nud, &np, &ual, &aal, &g, &gd, &s4, &elem, &w, &prev})
            b->release();
    }
};
}  // namespace

// two deterministic sums (partial rows 0, 1) -> host
static int sum2_dev(hbgpu_ctx* c, double* s0, double* s1) {
    launch_reduce_partials(c->partial.p, 2, c->red.p, 0, c->stream);
    TRY(check_launch(c));
    CK(c, cudaMemcpyAsync(c->h_red, c->red.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    *s0 = c->h_red[0];
    *s1 = c->h_red[1];
    return HBGPU_OK;
}

extern "C" int hbgpu_solve_time(hbgpu_ctx* c, const hbgpu_time_cfg* cfg, double period,
                                hbgpu_time_dirichlet_fn dirichlet, void* user, double* cycle_u,
                                double* cycle_p, hbgpu_time_result* result) {
    if (!c || !cfg || !dirichlet)
        return c ? fail(c, HBGPU_ERR_INVALID, "solve_time: null config or Dirichlet callback") : HBGPU_ERR_INVALID;
    if (c->N != 1)
        return fail(c, HBGPU_ERR_INVALID, "solve_time needs the N = 1 basis (hbgpu_set_basis(ctx, 1, period))");
    if (cfg->steps_per_cycle <= 0 || cfg->cycles <= 0 || !(period > 0.0))
        return fail(c, HBGPU_ERR_INVALID, "solve_time: steps_per_cycle, cycles and period must be positive");
    Timer total;
    cudaStream_t st = c->stream;
    const int nn = c->nn;
    const long n3 = 3L * nn;
    const bool steady = cfg->steady != 0;
    const double dt = period / double(cfg->steps_per_cycle);
    const double am = steady ? 0.0 : 0.5 * (3.0 - cfg->rho_inf) / (1.0 + cfg->rho_inf);
    const double af = steady ? 1.0 : 1.0 / (1.0 + cfg->rho_inf);
    const double gamma = steady ? 1.0 : 0.5 + am - af;
    hbgpu_time_result res{};
    TimeBufs tb;
    for (DBuf<double>* b : {&tb.u, &tb.ud, &tb.nu, &tb.nud, &tb.ual, &tb.aal, &tb.g, &tb.gd})
        CK(c, b->alloc(size_t(n3)));
    for (DBuf<double>* b : {&tb.p, &tb.np, &tb.w})
        CK(c, b->alloc(size_t(nn)));
    CK(c, tb.s4.alloc(size_t(nn) * 4));
    CK(c, tb.elem.alloc(size_t(c->ne) * 16));
    const int steps = cfg->steps_per_cycle;
    if (!steady && cfg->cycles > 1)
        CK(c, tb.prev.alloc(size_t(steps) * size_t(n3)));
    launch_nodal_volumes(c->geom.p, c->inc_ptr.p, c->inc_rec.p, nn, tb.w.p, st);

    // initial fields (time_solver.cpp:297-308): rest, outlet pressure level,
    // Dirichlet g(0), gdot(0)
    double wsum = 0.0, acc = 0.0;
    for (size_t k = 0; k < c->bc_patch.size(); ++k) {
        const double area = c->patches[size_t(c->bc_patch[k])].area;
        acc += area * (-c->h_h[k]);
        wsum += area;
    }
    const double p0 = std::isnan(cfg->initial_pressure) ? (wsum > 0.0 ? acc / wsum : 0.0) : cfg->initial_pressure;
    std::vector<double> hg(static_cast<size_t>(n3)), hgd(static_cast<size_t>(n3)), hu(static_cast<size_t>(n3), 0.0),
        hud(static_cast<size_t>(n3), 0.0), hp(static_cast<size_t>(nn), p0);
    dirichlet(0.0, hg.data(), hgd.data(), user);
    for (int a = 0; a < nn; ++a)
        if (c->dir_h[size_t(a)])
            for (int i = 0; i < 3; ++i) {
                hu[size_t(3 * a + i)] = hg[size_t(3 * a + i)];
                hud[size_t(3 * a + i)] = hgd[size_t(3 * a + i)];
            }
    CK(c, cudaMemcpy(tb.u.p, hu.data(), sizeof(double) * size_t(n3), cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(tb.ud.p, hud.data(), sizeof(double) * size_t(n3), cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(tb.p.p, hp.data(), sizeof(double) * size_t(nn), cudaMemcpyHostToDevice));
    if (c->partial.n < size_t(4) * kRedBlocks)
        CK(c, c->partial.alloc(size_t(kRedBlocks) * 1024));

    BoundaryArgs bargs = boundary_args(c, tb.s4.p, c->r.p);
    double omega_hat = 0.0;
    // one Newton-solved step to t_new (time_solver.cpp:354-455)
    auto newton_step = [&](double t_new, int step_index) -> int {
        dirichlet(t_new, hg.data(), hgd.data(), user);
        CK(c, cudaMemcpyAsync(tb.g.p, hg.data(), sizeof(double) * size_t(n3), cudaMemcpyHostToDevice, st));
        CK(c, cudaMemcpyAsync(tb.gd.p, hgd.data(), sizeof(double) * size_t(n3), cudaMemcpyHostToDevice, st));
        launch_time_predict(tb.u.p, tb.ud.p, tb.p.p, tb.g.p, tb.gd.p, c->dir.p, nn, steady ? 1 : 0, gamma, dt,
                            tb.nu.p, tb.nud.p, tb.np.p, st);
        double r0 = -1.0;
        const std::string where = " at step " + std::to_string(step_index);
        for (int k = 0; k <= cfg->max_newton_iters; ++k) {
            const double* eu = steady ? tb.nu.p : tb.ual.p;
            const double* ea = steady ? tb.nud.p : tb.aal.p;
            if (!steady) {
                launch_time_alpha(tb.u.p, tb.ud.p, tb.nu.p, tb.nud.p, nn, af, am, tb.ual.p, tb.aal.p, st);
                // acceleration scale of the current iterate
                launch_time_wnorm(tb.w.p, tb.ual.p, tb.aal.p, nn, c->partial.p, st);
                double su = 0.0, sa = 0.0;
                TRY(sum2_dev(c, &su, &sa));
                const double un = std::sqrt(su);
                omega_hat = un > 1e-14 ? std::sqrt(sa) / un : 0.0;
            } else {
                omega_hat = 0.0;
            }
            launch_time_residual(c->geom.p, c->conn.p, c->ne, c->inc_ptr.p, c->inc_rec.p, c->dir.p, nn, eu, ea,
                                 tb.np.p, c->rho, c->mu, omega_hat, tb.elem.p, c->r.p, st);
            if (c->nbnodes > 0) {
                launch_time_pack(eu, tb.np.p, nn, tb.s4.p, st);
                launch_boundary(bargs, st);
            }
            TRY(check_launch(c));
            double rn = 0.0;
            TRY(dot_dev(c, c->r.p, c->r.p, 4L * nn, &rn, true));
            if (!std::isfinite(rn))
                return fail(c, HBGPU_ERR_DIVERGENCE, "time solver diverged" + where);
            if (r0 < 0.0)
                r0 = rn;
            if (rn <= 1e-30 || rn <= r0 * std::pow(10.0, -cfg->newton_tol_orders))
                break;
            if (r0 > 0.0 && rn / r0 > 1e4)
                return fail(c, HBGPU_ERR_DIVERGENCE, "time solver diverged" + where);
            if (k == cfg->max_newton_iters)
                break;
            launch_time_tangent(c->geom.p, c->row_ptr.p, c->col_idx.p, c->inc_ptr.p, c->inc_rec.p, c->dir.p, nn,
                                eu, c->rho, c->mu, omega_hat, am, steady ? 1.0 : af * gamma * dt, c->pvals.p, st);
            TRY(check_launch(c));
            c->p_valid = true;
            c->inv_valid = false;
            TRY(jacobi_dev(c, nullptr));
            hbgpu_krylov_result kr{};
            TRY(gmres_dev(c, c->r.p, c->inv.p, &cfg->krylov, c->x.p, &kr, nullptr, 0));
            if (kr.status == 2)
                return fail(c, HBGPU_ERR_STAGNATION, "time solver GMRES stagnated" + where);
            res.total_newton_iters += 1;
            launch_time_update(c->x.p, c->dir.p, nn, steady ? 1 : 0, gamma * dt, tb.nu.p, tb.nud.p, tb.np.p, st);
            TRY(check_launch(c));
        }
        res.omega_hat_last = omega_hat;
        std::swap(tb.u, tb.nu);
        std::swap(tb.ud, tb.nud);
        std::swap(tb.p, tb.np);
        return HBGPU_OK;
    };
    auto finish = [&](int code) {
        res.total_seconds = total.seconds();
        if (result)
            *result = res;
        return code;
    };

    if (steady) {
        const int s = newton_step(0.0, 0);
        if (s != HBGPU_OK)
            return finish(s);
        if (cycle_u)
            CK(c, cudaMemcpy(cycle_u, tb.u.p, sizeof(double) * size_t(n3), cudaMemcpyDeviceToHost));
        if (cycle_p)
            CK(c, cudaMemcpy(cycle_p, tb.p.p, sizeof(double) * size_t(nn), cudaMemcpyDeviceToHost));
        res.total_steps = 1;
        return finish(HBGPU_OK);
    }
    double diff2 = 0.0, norm2acc = 0.0;
    for (int cycle = 0; cycle < cfg->cycles; ++cycle) {
        const bool last = cycle == cfg->cycles - 1;
        if (last) {
            if (cycle_u)
                CK(c, cudaMemcpy(cycle_u, tb.u.p, sizeof(double) * size_t(n3), cudaMemcpyDeviceToHost));
            if (cycle_p)
                CK(c, cudaMemcpy(cycle_p, tb.p.p, sizeof(double) * size_t(nn), cudaMemcpyDeviceToHost));
        }
        if (cycle == cfg->cycles - 1 || cycle == cfg->cycles - 2) {
            diff2 = 0.0;
            norm2acc = 0.0;
        }
        for (int j = 0; j < steps; ++j) {
            const double t_new = (double(cycle) * steps + j + 1) * dt;
            const int s = newton_step(t_new, cycle * steps + j);
            if (s != HBGPU_OK)
                return finish(s);
            res.total_steps += 1;
            if (tb.prev.p) {
                launch_time_cycle(tb.u.p, tb.prev.p + size_t(j) * size_t(n3), n3, cycle > 0 ? 1 : 0, c->partial.p,
                                  st);
                if (cycle > 0) {
                    double d2 = 0.0, u2 = 0.0;
                    TRY(sum2_dev(c, &d2, &u2));
                    diff2 += d2;
                    norm2acc += u2;
                }
            }
            if (last) {
                if (cycle_u)
                    CK(c, cudaMemcpy(cycle_u + size_t(j + 1) * size_t(n3), tb.u.p, sizeof(double) * size_t(n3),
                                     cudaMemcpyDeviceToHost));
                if (cycle_p)
                    CK(c, cudaMemcpy(cycle_p + size_t(j + 1) * size_t(nn), tb.p.p, sizeof(double) * size_t(nn),
                                     cudaMemcpyDeviceToHost));
            }
        }
        if (cycle > 0)
            res.cycle_change = norm2acc > 0.0 ? std::sqrt(diff2 / norm2acc) : 0.0;
    }
    return finish(HBGPU_OK);
}

extern "C" int hbgpu_time_residual(hbgpu_ctx* c, const double* u, const double* udot, const double* p,
                                   double omega_hat, double* r) {
    if (!c || !u || !udot || !p || !r)
        return c ? fail(c, HBGPU_ERR_INVALID, "time_residual: null buffer") : HBGPU_ERR_INVALID;
    if (c->N != 1)
        return fail(c, HBGPU_ERR_INVALID, "time_residual needs the N = 1 basis");
    const int nn = c->nn;
    cudaStream_t st = c->stream;
    TimeBufs tb;
    for (DBuf<double>* b : {&tb.u, &tb.ud})
        CK(c, b->alloc(size_t(nn) * 3));
    CK(c, tb.p.alloc(size_t(nn)));
    CK(c, tb.s4.alloc(size_t(nn) * 4));
    CK(c, tb.elem.alloc(size_t(c->ne) * 16));
    CK(c, cudaMemcpyAsync(tb.u.p, u, sizeof(double) * size_t(nn) * 3, cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(tb.ud.p, udot, sizeof(double) * size_t(nn) * 3, cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(tb.p.p, p, sizeof(double) * size_t(nn), cudaMemcpyHostToDevice, st));
    launch_time_residual(c->geom.p, c->conn.p, c->ne, c->inc_ptr.p, c->inc_rec.p, c->dir.p, nn, tb.u.p, tb.ud.p,
                         tb.p.p, c->rho, c->mu, omega_hat, tb.elem.p, c->r.p, st);
    if (c->nbnodes > 0) {
        launch_time_pack(tb.u.p, tb.p.p, nn, tb.s4.p, st);
        launch_boundary(boundary_args(c, tb.s4.p, c->r.p), st);
    }
    TRY(check_launch(c));
    CK(c, cudaMemcpyAsync(r, c->r.p, sizeof(double) * size_t(nn) * 4, cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    return HBGPU_OK;
}

extern "C" int hbgpu_time_tangent(hbgpu_ctx* c, const double* u, double omega_hat, double am, double fg,
                                  double* pvals) {
    if (!c || !u)
        return c ? fail(c, HBGPU_ERR_INVALID, "time_tangent: null buffer") : HBGPU_ERR_INVALID;
    if (c->N != 1)
        return fail(c, HBGPU_ERR_INVALID, "time_tangent needs the N = 1 basis");
    const int nn = c->nn;
    cudaStream_t st = c->stream;
    TimeBufs tb;
    CK(c, tb.u.alloc(size_t(nn) * 3));
    CK(c, cudaMemcpyAsync(tb.u.p, u, sizeof(double) * size_t(nn) * 3, cudaMemcpyHostToDevice, st));
    launch_time_tangent(c->geom.p, c->row_ptr.p, c->col_idx.p, c->inc_ptr.p, c->inc_rec.p, c->dir.p, nn, tb.u.p,
                        c->rho, c->mu, omega_hat, am, fg, c->pvals.p, st);
    TRY(check_launch(c));
    c->p_valid = true;
    c->inv_valid = false;
    if (pvals)
        CK(c, cudaMemcpyAsync(pvals, c->pvals.p, sizeof(double) * size_t(c->nnz) * 8, cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    return HBGPU_OK;
}
