// Time-domain (generalized-alpha) GLS operators on the GPU — the reference's
// time-stepping solver (src/time_solver.cpp), the comparison baseline of the
// paper, run on the same N = 1 machinery as the harmonic-balance path
// (L-matvec with H = 0, Jacobi, the device-resident GMRES).
//
//   time_residual  time_solver.cpp:58-166   element pass + row gather in
//                  element order, then the shared boundary kernel (steady
//                  outlet traction h[0] + backflow) and Dirichlet rows
//   time_tangent   time_solver.cpp:172-254  row-owned: each block row of P
//                  sums its elements' (a, b) blocks in element order, the
//                  reference's scatter order
//   tau_hat        time_solver.cpp:34-43    (omega_hat^2 + u.xi.u + 3 nu^2 xi:xi)^-1/2
//
// FP64, deterministic (no atomics).  Geometry: the reference's 22-double
// ElementGeometry records (gradN 12, V, xi row-major 9).
#include "hbgpu_internal.h"

namespace hbgpu {

namespace {
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

__device__ __forceinline__ double shape_q(int q, int a) { return q == a ? kQA : kQB; }

__device__ __forceinline__ double tau_hat(const double* __restrict__ g, const double u[3], double nu,
                                          double omega_hat) {
    double conv = 0.0, xx = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double x = g[13 + 3 * i + j];
            conv += u[i] * x * u[j];
            xx += x * x;
        }
    return 1.0 / sqrt(omega_hat * omega_hat + conv + 3.0 * nu * nu * xx);
}
}  // namespace

// Element pass of time_residual: thread per element, its 16 contributions
// (node a: momentum 0..2, continuity 3) into out[e*16 + a*4 + c].
// u, udot: node*3+i;  p: node.
__global__ void time_residual_elem_kernel(const double* __restrict__ geom, const int4* __restrict__ conn,
                                          int ne, const double* __restrict__ u,
                                          const double* __restrict__ udot, const double* __restrict__ p,
                                          double rho, double mu, double omega_hat,
                                          double* __restrict__ out) {
    const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne)
        return;
    const double* g = geom + 22 * e;
    const int4 c4 = conn[e];
    const int nd[4] = {c4.x, c4.y, c4.z, c4.w};
    const double nu = mu / rho, w = g[12] / 4.0;
    double un[4][3], an[4][3], pn[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            un[a][i] = u[3L * nd[a] + i];
            an[a][i] = udot[3L * nd[a] + i];
        }
        pn[a] = p[nd[a]];
    }
    double gradu[3][3] = {}, gradp[3] = {};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
#pragma unroll
            for (int j = 0; j < 3; ++j)
                gradu[i][j] += g[3 * a + j] * un[a][i];
            gradp[i] += g[3 * a + i] * pn[a];
        }
    const double divu = gradu[0][0] + gradu[1][1] + gradu[2][2];
    double r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
        r[k] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double uq[3] = {}, aq[3] = {}, pq = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const double sa = shape_q(q, a);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                uq[i] += sa * un[a][i];
                aq[i] += sa * an[a][i];
            }
            pq += sa * pn[a];
        }
        const double th = tau_hat(g, uq, nu, omega_hat);
        double conv[3], lq[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double cv = 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j)
                cv += uq[j] * gradu[i][j];
            conv[i] = cv;
            lq[i] = rho * aq[i] + rho * cv + gradp[i];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const double sa = shape_q(q, a);
            double adv = 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j)
                adv += uq[j] * g[3 * a + j];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                double visc = 0.0;
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    visc += g[3 * a + j] * gradu[i][j];
                r[a * 4 + i] += w * (rho * sa * (aq[i] + conv[i]) - g[3 * a + i] * pq + mu * visc +
                                     adv * th * lq[i]);
            }
            double pspg = 0.0;
#pragma unroll
            for (int i = 0; i < 3; ++i)
                pspg += g[3 * a + i] * th * lq[i];
            r[a * 4 + 3] += w * (sa * divu + pspg / rho);
        }
    }
    double* o = out + 16 * e;
#pragma unroll
    for (int k = 0; k < 16; ++k)
        o[k] = r[k];
}

// Row gather: r[A*4+c] = sum over A's incidences (element order) of the
// element contributions; Dirichlet velocity rows zero (time_solver.cpp:162-165;
// the boundary kernel skips them, so zeroing first is equivalent).
__global__ void time_residual_rows_kernel(const double* __restrict__ elem, const int* __restrict__ inc_ptr,
                                          const int4* __restrict__ rec, const uint8_t* __restrict__ dir,
                                          int nn, double* __restrict__ r) {
    const int A = blockIdx.x * blockDim.x + threadIdx.x;
    if (A >= nn)
        return;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int ii = inc_ptr[A]; ii < inc_ptr[A + 1]; ++ii) {
        const int4 r1 = rec[2 * ii + 1];
        const long e = r1.x & 0x3FFFFFFF;
        const int la = (unsigned)r1.x >> 30;
        const double* o = elem + 16 * e + 4 * la;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            acc[c] += o[c];
    }
    const bool fix = dir[A] != 0;
#pragma unroll
    for (int c = 0; c < 4; ++c)
        r[4L * A + c] = (fix && c < 3) ? 0.0 : acc[c];
}

void launch_time_residual(const double* geom, const int4* conn, int ne, const int* inc_ptr, const int4* rec,
                          const uint8_t* dir, int nn, const double* u, const double* udot, const double* p,
                          double rho, double mu, double omega_hat, double* elem, double* r, cudaStream_t st) {
    if (ne <= 0)
        return;
    note_launch();
    time_residual_elem_kernel<<<(ne + 127) / 128, 128, 0, st>>>(geom, conn, ne, u, udot, p, rho, mu, omega_hat,
                                                                 elem);
    note_launch();
    time_residual_rows_kernel<<<(nn + 127) / 128, 128, 0, st>>>(elem, inc_ptr, rec, dir, nn, r);
}

// time_tangent, row-owned: thread per block row A.  For each incidence
// (element e, local index a) in element order, the element's blocks (a, b),
// b = 0..3, are formed exactly as the reference forms K, G, D, L
// (constant part, then the quadrature sum) and added to the row's blocks
// with the Dirichlet masks (K: both free, G: row free, D: column free, L:
// always); identity K on Dirichlet diagonals.  P: N = 1, vals[blk*8 + slot].
__global__ void time_tangent_rows_kernel(const double* __restrict__ geom, const int* __restrict__ row_ptr,
                                         const int* __restrict__ col_idx, const int* __restrict__ inc_ptr,
                                         const int4* __restrict__ rec, const uint8_t* __restrict__ dir,
                                         int nn, const double* __restrict__ u, double rho, double mu,
                                         double omega_hat, double am, double fg, double* __restrict__ vals) {
    const int A = blockIdx.x * blockDim.x + threadIdx.x;
    if (A >= nn)
        return;
    const int k0 = row_ptr[A], k1 = row_ptr[A + 1];
    for (long k = (long)k0 * 8; k < (long)k1 * 8; ++k)
        vals[k] = 0.0;
    const double nu = mu / rho;
    const bool afix = dir[A] != 0;
    for (int ii = inc_ptr[A]; ii < inc_ptr[A + 1]; ++ii) {
        const int4 c4 = rec[2 * ii];
        const int4 r1 = rec[2 * ii + 1];
        const long e = r1.x & 0x3FFFFFFF;
        const int a = (unsigned)r1.x >> 30;
        const unsigned cols = (unsigned)r1.y;
        const int nd[4] = {c4.x, c4.y, c4.z, c4.w};
        const double* g = geom + 22 * e;
        const double V = g[12], w = V / 4.0;
        double un[4][3];
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int i = 0; i < 3; ++i)
                un[b][i] = u[3L * nd[b] + i];
        double K[4], G[4][3], D[4][3], L[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            double gg = 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j)
                gg += g[3 * a + j] * g[3 * b + j];
            const double mab = (a == b) ? V / 10.0 : V / 20.0;  // element_mass(g, 1.0)
            K[b] = 0.0 + (am * rho * mab + fg * mu * V * gg);
            L[b] = 0.0;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                G[b][i] = 0.0 + -g[3 * a + i] * V / 4.0;
                D[b][i] = 0.0 + fg * g[3 * b + i] * V / 4.0;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double uq[3] = {};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const double sb = shape_q(q, b);
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    uq[i] += sb * un[b][i];
            }
            const double th = tau_hat(g, uq, nu, omega_hat);
            double adv[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                adv[b] = 0.0;
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    adv[b] += uq[j] * g[3 * b + j];
            }
            const double sa = shape_q(q, a);
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const double sb = shape_q(q, b);
                K[b] += w * (fg * rho * (sa * adv[b] + adv[a] * th * adv[b]) + am * rho * adv[a] * th * sb);
                double gg = 0.0;
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    gg += g[3 * a + j] * g[3 * b + j];
                L[b] += w * gg * th / rho;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    G[b][i] += w * adv[a] * th * g[3 * b + i];
                    D[b][i] += w * g[3 * a + i] * th * (am * sb + fg * adv[b]);
                }
            }
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const bool bfix = dir[nd[b]] != 0;
            double* v = vals + 8L * (k0 + (int)((cols >> (8 * b)) & 0xFFu));
            if (!afix && !bfix)
                v[0] += K[b];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                if (!afix)
                    v[1 + i] += G[b][i];
                if (!bfix)
                    v[4 + i] += D[b][i];
            }
            v[7] += L[b];
        }
    }
    if (afix)
        for (int k = k0; k < k1; ++k)
            if (col_idx[k] == A)
                vals[8L * k] = 1.0;
}

void launch_time_tangent(const double* geom, const int* row_ptr, const int* col_idx, const int* inc_ptr,
                         const int4* rec, const uint8_t* dir, int nn, const double* u, double rho, double mu,
                         double omega_hat, double am, double fg, double* vals, cudaStream_t st) {
    if (nn <= 0)
        return;
    note_launch();
    time_tangent_rows_kernel<<<(nn + 63) / 64, 64, 0, st>>>(geom, row_ptr, col_idx, inc_ptr, rec, dir, nn, u, rho,
                                                            mu, omega_hat, am, fg, vals);
}

// ---------------------------------------------------------------- stepping helpers
// Generalized-alpha predictor (time_solver.cpp:359-380): next = state with
// udot scaled by (gamma-1)/gamma (unsteady), Dirichlet nodes landing on g(t).
__global__ void time_predict_kernel(const double* __restrict__ u, const double* __restrict__ ud,
                                    const double* __restrict__ p, const double* __restrict__ g,
                                    const double* __restrict__ gd, const uint8_t* __restrict__ dir, int nn,
                                    int steady, double gamma, double dt, double* __restrict__ nu_,
                                    double* __restrict__ nud, double* __restrict__ np) {
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= 3L * nn)
        return;
    const long A = k / 3;
    double un = u[k], udn = steady ? ud[k] : ud[k] * ((gamma - 1.0) / gamma);
    if (dir[A]) {
        if (steady) {
            un = g[k];
            udn = 0.0;
        } else {
            udn = (g[k] - u[k]) / (gamma * dt) - (1.0 - gamma) / gamma * ud[k];
            un = g[k];
        }
    }
    nu_[k] = un;
    nud[k] = udn;
    if (k % 3 == 0)
        np[A] = p[A];
}

// ual = u + af (next.u - u), aal = udot + am (next.udot - udot)
__global__ void time_alpha_kernel(const double* __restrict__ u, const double* __restrict__ ud,
                                  const double* __restrict__ nu_, const double* __restrict__ nud, long n3,
                                  double af, double am, double* __restrict__ ual, double* __restrict__ aal) {
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n3)
        return;
    ual[k] = u[k] + af * (nu_[k] - u[k]);
    aal[k] = ud[k] + am * (nud[k] - ud[k]);
}

// Newton update (time_solver.cpp:438-453): free velocity dofs take -dv on
// udot (and -gamma dt dv on u), or -dv on u (steady); every pressure -x_p.
__global__ void time_update_kernel(const double* __restrict__ x, const uint8_t* __restrict__ dir, int nn,
                                   int steady, double gdt, double* __restrict__ nu_, double* __restrict__ nud,
                                   double* __restrict__ np) {
    const int A = blockIdx.x * blockDim.x + threadIdx.x;
    if (A >= nn)
        return;
    if (!dir[A])
        for (int i = 0; i < 3; ++i) {
            const double dv = x[4L * A + i];
            if (steady) {
                nu_[3L * A + i] -= dv;
            } else {
                nud[3L * A + i] -= dv;
                nu_[3L * A + i] -= gdt * dv;
            }
        }
    np[A] -= x[4L * A + 3];
}

// s4[A*4+c] = (u_A, p_A): the N = 1 state layout the boundary kernel reads
__global__ void time_pack_kernel(const double* __restrict__ u, const double* __restrict__ p, int nn,
                                 double* __restrict__ s4) {
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= 4L * nn)
        return;
    const long A = k >> 2;
    const int c = (int)(k & 3);
    s4[k] = c < 3 ? u[3 * A + c] : p[A];
}

// Per-CTA partials of sum_A w_A |f_A|^2 for up to two node fields (row 0: f0,
// row 1: f1), and of the cycle-to-cycle change sums (rows 2, 3).
__global__ void time_wnorm_kernel(const double* __restrict__ w, const double* __restrict__ f0,
                                  const double* __restrict__ f1, int nn, double* partial) {
    __shared__ double red[2][8];
    double s0 = 0.0, s1 = 0.0;
    for (long A = (long)blockIdx.x * blockDim.x + threadIdx.x; A < nn; A += (long)gridDim.x * blockDim.x) {
        double m0 = 0.0, m1 = 0.0;
        for (int i = 0; i < 3; ++i) {
            const double x0 = f0[3 * A + i];
            m0 += x0 * x0;
            if (f1) {
                const double x1 = f1[3 * A + i];
                m1 += x1 * x1;
            }
        }
        s0 += w[A] * m0;
        s1 += w[A] * m1;
    }
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_down_sync(0xffffffffu, s0, o);
        s1 += __shfl_down_sync(0xffffffffu, s1, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = s0;
        red[1][threadIdx.x >> 5] = s1;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k)
            t += red[threadIdx.x][k];
        partial[(long)threadIdx.x * kRedBlocks + blockIdx.x] = t;
    }
}

// cycle change: partial rows 0/1 of sum (f - buf)^2 and sum f^2; buf <- f
__global__ void time_cycle_kernel(const double* __restrict__ f, double* __restrict__ buf, long n3, int accumulate,
                                  double* partial) {
    __shared__ double red[2][8];
    double s0 = 0.0, s1 = 0.0;
    for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n3; k += (long)gridDim.x * blockDim.x) {
        const double v = f[k];
        if (accumulate) {
            const double d = v - buf[k];
            s0 += d * d;
            s1 += v * v;
        }
        buf[k] = v;
    }
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_down_sync(0xffffffffu, s0, o);
        s1 += __shfl_down_sync(0xffffffffu, s1, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = s0;
        red[1][threadIdx.x >> 5] = s1;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k)
            t += red[threadIdx.x][k];
        partial[(long)threadIdx.x * kRedBlocks + blockIdx.x] = t;
    }
}

// nodal_volumes (mesh.cpp:226-236): w_A = sum of V_e / 4 over A's elements, element order
__global__ void nodal_volumes_kernel(const double* __restrict__ geom, const int* __restrict__ inc_ptr,
                                     const int4* __restrict__ rec, int nn, double* __restrict__ w) {
    const int A = blockIdx.x * blockDim.x + threadIdx.x;
    if (A >= nn)
        return;
    double s = 0.0;
    for (int ii = inc_ptr[A]; ii < inc_ptr[A + 1]; ++ii)
        s += geom[22L * (rec[2 * ii + 1].x & 0x3FFFFFFF) + 12] / 4.0;
    w[A] = s;
}
void launch_nodal_volumes(const double* geom, const int* inc_ptr, const int4* rec, int nn, double* w,
                          cudaStream_t st) {
    note_launch();
    nodal_volumes_kernel<<<(nn + 255) / 256, 256, 0, st>>>(geom, inc_ptr, rec, nn, w);
}

void launch_time_predict(const double* u, const double* ud, const double* p, const double* g, const double* gd,
                         const uint8_t* dir, int nn, int steady, double gamma, double dt, double* nu_, double* nud,
                         double* np, cudaStream_t st) {
    note_launch();
    time_predict_kernel<<<(int)((3L * nn + 255) / 256), 256, 0, st>>>(u, ud, p, g, gd, dir, nn, steady, gamma, dt,
                                                                    nu_, nud, np);
}
void launch_time_alpha(const double* u, const double* ud, const double* nu_, const double* nud, int nn,
                       double af, double am, double* ual, double* aal, cudaStream_t st) {
    note_launch();
    time_alpha_kernel<<<(int)((3L * nn + 255) / 256), 256, 0, st>>>(u, ud, nu_, nud, 3L * nn, af, am, ual, aal);
}
void launch_time_update(const double* x, const uint8_t* dir, int nn, int steady, double gdt, double* nu_,
                        double* nud, double* np, cudaStream_t st) {
    note_launch();
    time_update_kernel<<<(nn + 255) / 256, 256, 0, st>>>(x, dir, nn, steady, gdt, nu_, nud, np);
}
void launch_time_pack(const double* u, const double* p, int nn, double* s4, cudaStream_t st) {
    note_launch();
    time_pack_kernel<<<(int)((4L * nn + 255) / 256), 256, 0, st>>>(u, p, nn, s4);
}
void launch_time_wnorm(const double* w, const double* f0, const double* f1, int nn, double* partial,
                       cudaStream_t st) {
    note_launch();
    time_wnorm_kernel<<<kRedBlocks, 256, 0, st>>>(w, f0, f1, nn, partial);
}
void launch_time_cycle(const double* f, double* buf, long n3, int accumulate, double* partial, cudaStream_t st) {
    note_launch();
    time_cycle_kernel<<<kRedBlocks, 256, 0, st>>>(f, buf, n3, accumulate, partial);
}

}  // namespace hbgpu
