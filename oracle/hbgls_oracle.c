/* hbgls_oracle.c — plain-C CPU restatement of the reference HB-GLS hot path.
 * TEST INFRASTRUCTURE ONLY; see hbgls_oracle.h for layouts and pinning.
 *
 * Written per (element, time sample): the HB-GLS element operators are
 * diagonal in time once the nodal pseudo-spectral derivative H*u is known
 * (assembly.cpp:453-463), so every element/sample pair is independent.  This
 * is the same decomposition the CUDA kernels use, spelled out serially.
 */
#define _POSIX_C_SOURCE 200112L
#include "hbgls_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* 4-point tet rule, assembly.cpp:15-20; weight V/4 (assembly.cpp:154). */
static const double QA = 0.5854101966249684544613761;
static const double QB = 0.1381966011250105151795414;
static double tet_shape(int q, int a) { return q == a ? QA : QB; }
/* 3-point triangle rule, assembly.cpp:23-25; weight area/3 (:384). */
static double tri_shape(int q, int a) { return q == a ? 2.0 / 3.0 : 1.0 / 6.0; }

#define GN(g, a, j) ((g)[3 * (a) + (j)])
#define GV(g) ((g)[12])
#define GXI(g, i, j) ((g)[13 + 3 * (i) + (j)])

/* ---------------------------------------------------------------- spectral */

void hbo_h_dense(int modes, double period, double* H) {
    /* H = real(E^{-1} Omega E), E(l,k) = e^{-2 pi i l k/N}/N, Omega_ll = i*omega*m(l),
     * m(l) = l for l < M else l - N   (spectral.cpp:14-15,236-256). */
    const int M = modes, N = 2 * modes - 1;
    const double two_pi = 6.283185307179586476925286766559;
    const double omega = two_pi / period;
    for (int j = 0; j < N; ++j)
        for (int k = 0; k < N; ++k) {
            double acc = 0.0;
            for (int l = 0; l < N; ++l) {
                const double m = (double)(l < M ? l : l - N);
                /* real part of e^{i a} * (i w m) * e^{-i b}/N = -w m sin(a - b)/N */
                const double a = two_pi * (double)j * (double)l / (double)N;
                const double b = two_pi * (double)l * (double)k / (double)N;
                acc += -omega * m * (sin(a) * cos(b) - cos(a) * sin(b)) / (double)N;
            }
            H[j * N + k] = acc;
        }
}

/* ---------------------------------------------------------------- geometry */

int hbo_geometry(int nn, const double* xyz, int ne, const int* conn, double* geom) {
    (void)nn;
    for (int e = 0; e < ne; ++e) {
        const double* x0 = xyz + 3 * conn[4 * e + 0];
        double c[3][3]; /* columns x1-x0, x2-x0, x3-x0 (mesh.cpp:168) */
        for (int k = 0; k < 3; ++k)
            for (int i = 0; i < 3; ++i)
                c[k][i] = xyz[3 * conn[4 * e + 1 + k] + i] - x0[i];
        const double det = c[0][0] * (c[1][1] * c[2][2] - c[1][2] * c[2][1]) -
                           c[1][0] * (c[0][1] * c[2][2] - c[0][2] * c[2][1]) +
                           c[2][0] * (c[0][1] * c[1][2] - c[0][2] * c[1][1]);
        double* g = geom + 22 * (size_t)e;
        GV(g) = det / 6.0;
        if (!(GV(g) > 0.0))
            return -1;
        /* rows of J^{-1}: cross products of the other two columns over det */
        double r[3][3];
        for (int k = 0; k < 3; ++k) {
            const double* u = c[(k + 1) % 3];
            const double* v = c[(k + 2) % 3];
            r[k][0] = (u[1] * v[2] - u[2] * v[1]) / det;
            r[k][1] = (u[2] * v[0] - u[0] * v[2]) / det;
            r[k][2] = (u[0] * v[1] - u[1] * v[0]) / det;
        }
        for (int i = 0; i < 3; ++i) {
            GN(g, 1, i) = r[0][i];
            GN(g, 2, i) = r[1][i];
            GN(g, 3, i) = r[2][i];
            GN(g, 0, i) = -(r[0][i] + r[1][i] + r[2][i]);
        }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                GXI(g, i, j) = r[0][i] * r[0][j] + r[1][i] * r[1][j] + r[2][i] * r[2][j];
    }
    return 0;
}

/* ---------------------------------------------------------------- pattern */

static int cmp_int(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

int hbo_pattern(int nn, int ne, const int* conn, int* row_ptr, int* col_idx) {
    /* CSR over element adjacency, diagonal always present, columns sorted
     * and unique per row (linalg.cpp:10-30). */
    int* cnt = calloc((size_t)nn + 1, sizeof(int));
    for (int e = 0; e < ne; ++e)
        for (int a = 0; a < 4; ++a)
            cnt[conn[4 * e + a] + 1] += 4;
    for (int a = 0; a < nn; ++a)
        cnt[a + 1] += cnt[a] + 1; /* +1 for the forced diagonal */
    int* buf = malloc(sizeof(int) * (size_t)(cnt[nn] > 0 ? cnt[nn] : 1));
    int* fill = malloc(sizeof(int) * (size_t)(nn > 0 ? nn : 1));
    for (int a = 0; a < nn; ++a) {
        fill[a] = cnt[a];
        buf[fill[a]++] = a;
    }
    for (int e = 0; e < ne; ++e)
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                const int A = conn[4 * e + a];
                buf[fill[A]++] = conn[4 * e + b];
            }
    int nnz = 0;
    if (row_ptr)
        row_ptr[0] = 0;
    for (int a = 0; a < nn; ++a) {
        int* row = buf + cnt[a];
        const int len = cnt[a + 1] - cnt[a];
        qsort(row, (size_t)len, sizeof(int), cmp_int);
        int u = 0;
        for (int k = 0; k < len; ++k)
            if (k == 0 || row[k] != row[k - 1])
                row[u++] = row[k];
        if (col_idx)
            memcpy(col_idx + nnz, row, sizeof(int) * (size_t)u);
        nnz += u;
        if (row_ptr)
            row_ptr[a + 1] = nnz;
    }
    free(cnt);
    free(buf);
    free(fill);
    return nnz;
}

int hbo_find(const int* row_ptr, const int* col_idx, int a, int b) {
    int lo = row_ptr[a], hi = row_ptr[a + 1];
    while (lo < hi) {
        const int mid = lo + (hi - lo) / 2;
        if (col_idx[mid] < b)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < row_ptr[a + 1] && col_idx[lo] == b) ? lo : -1;
}

/* ---------------------------------------------------------------- tau */

/* tau = (u.xi.u + C_I nu^2 xi:xi)^(-1/2), C_I = 3 (assembly.hpp:15, assembly.cpp:43-56) */
static int tau_of(const double* g, const double u[3], double nu, double* tau) {
    double xx = 0.0, conv = 0.0;
    for (int k = 0; k < 9; ++k)
        xx += g[13 + k] * g[13 + k];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            conv += u[i] * GXI(g, i, j) * u[j];
    const double arg = conv + 3.0 * nu * nu * xx;
    if (!(arg > 0.0))
        return -1;
    *tau = 1.0 / sqrt(arg);
    return 0;
}

static void apply_h(int N, const double* H, const double* in, double* out) {
    for (int n = 0; n < N; ++n) {
        double acc = 0.0;
        for (int m = 0; m < N; ++m)
            acc += H[n * N + m] * in[m];
        out[n] = acc;
    }
}

/* ---------------------------------------------------------------- residual */

/* One element at one time sample: accumulates r_m[a][i], r_c[a], s[a][i]
 * (assembly.cpp:141-263, element_residual). */
static int element_residual_n(const hbo_problem* p, const double* g, const double u[4][3],
                              const double pr[4], const double hu[4][3], double rm[4][3],
                              double rc[4], double s[4][3]) {
    const double V = GV(g), rho = p->rho, mu = p->mu, nu = mu / rho, w = V / 4.0;
    double gu[3][3] = {{0}}, gp[3] = {0};
    for (int a = 0; a < 4; ++a)
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j)
                gu[i][j] += GN(g, a, j) * u[a][i];
            gp[i] += GN(g, a, i) * pr[a];
        }
    const double div = gu[0][0] + gu[1][1] + gu[2][2];
    double psum = 0.0;
    for (int b = 0; b < 4; ++b)
        psum += pr[b];
    /* Galerkin rows with constant gradients (assembly.cpp:156-192) */
    for (int a = 0; a < 4; ++a) {
        for (int i = 0; i < 3; ++i) {
            double v = 0.0;
            for (int j = 0; j < 3; ++j)
                v += mu * V * GN(g, a, j) * gu[i][j];
            v += -GN(g, a, i) * (V / 4.0) * psum;
            for (int b = 0; b < 4; ++b)
                v += rho * (a == b ? V / 10.0 : V / 20.0) * hu[b][i];
            rm[a][i] += v;
        }
        rc[a] += w * div;
    }
    double tau_mean = 0.0;
    if (p->tau_mode == 1) {
        double um[3] = {0, 0, 0};
        for (int a = 0; a < 4; ++a)
            for (int i = 0; i < 3; ++i)
                um[i] += 0.25 * u[a][i];
        if (tau_of(g, um, nu, &tau_mean))
            return -1;
    }
    for (int q = 0; q < 4; ++q) {
        double uq[3] = {0, 0, 0}, huq[3] = {0, 0, 0};
        for (int i = 0; i < 3; ++i)
            for (int a = 0; a < 4; ++a) {
                uq[i] += tet_shape(q, a) * u[a][i];
                huq[i] += tet_shape(q, a) * hu[a][i];
            }
        double tau = tau_mean;
        if (p->tau_mode == 0 && tau_of(g, uq, nu, &tau))
            return -1;
        double conv[3], L[3], adv[4];
        for (int i = 0; i < 3; ++i) {
            conv[i] = uq[0] * gu[i][0] + uq[1] * gu[i][1] + uq[2] * gu[i][2];
            L[i] = rho * huq[i] + rho * conv[i] + gp[i]; /* strong residual, :213-224 */
        }
        for (int a = 0; a < 4; ++a)
            adv[a] = uq[0] * GN(g, a, 0) + uq[1] * GN(g, a, 1) + uq[2] * GN(g, a, 2);
        for (int a = 0; a < 4; ++a) {
            const double sa = tet_shape(q, a);
            double cont = 0.0;
            for (int i = 0; i < 3; ++i) {
                const double tl = tau * L[i];
                rm[a][i] += w * (rho * sa * conv[i] + adv[a] * tl);
                s[a][i] += w * sa * tl;
                cont += GN(g, a, i) * tau * L[i];
            }
            rc[a] += w * cont / rho;
        }
    }
    return 0;
}

/* Neumann traction + backflow for every listed facet (assembly.cpp:376-413). */
static void boundary_terms(const hbo_problem* p, const double* state, double* r) {
    const int N = p->N;
    for (int f = 0; f < p->nfac; ++f) {
        const int* fac = p->fac + 3 * f;
        const double* nv = p->fnormal + 3 * f;
        const double* h = p->h + (size_t)p->fbc[f] * N;
        const double w = p->farea[f] / 3.0;
        for (int q = 0; q < 3; ++q)
            for (int n = 0; n < N; ++n) {
                double uq[3] = {0, 0, 0};
                for (int a = 0; a < 3; ++a)
                    for (int i = 0; i < 3; ++i)
                        uq[i] += tri_shape(q, a) * state[((size_t)fac[a] * 4 + i) * N + n];
                const double un = uq[0] * nv[0] + uq[1] * nv[1] + uq[2] * nv[2];
                const double neg = un < 0.0 ? un : 0.0;
                for (int a = 0; a < 3; ++a)
                    for (int i = 0; i < 3; ++i)
                        r[((size_t)fac[a] * 4 + i) * N + n] +=
                            w * tri_shape(q, a) *
                            (-h[n] * nv[i] - 0.5 * p->rho * p->beta * neg * uq[i]);
            }
    }
}

static int neumann_entries(const hbo_problem* p) {
    int ne = 0;
    for (int f = 0; f < p->nfac; ++f)
        if (p->fbc[f] + 1 > ne)
            ne = p->fbc[f] + 1;
    return ne;
}

/* Resistance outlets (see hbgls_oracle.h): flux of `v` (layout (node*4+i)*N+n)
 * through Neumann entry k at sample n, 3-point facet rule; free_only: only the
 * non-Dirichlet nodes' values count (the tangent's masked columns). */
static double entry_flux(const hbo_problem* p, int k, const double* v, int n, int free_only) {
    const int N = p->N;
    double Q = 0.0;
    for (int f = 0; f < p->nfac; ++f) {
        if (p->fbc[f] != k)
            continue;
        const int* fac = p->fac + 3 * f;
        const double* nv = p->fnormal + 3 * f;
        const double w = p->farea[f] / 3.0;
        for (int q = 0; q < 3; ++q) {
            double un = 0.0;
            for (int a = 0; a < 3; ++a) {
                if (free_only && p->dirichlet[fac[a]])
                    continue;
                for (int i = 0; i < 3; ++i)
                    un += tri_shape(q, a) * v[((size_t)fac[a] * 4 + i) * N + n] * nv[i];
            }
            Q += w * un;
        }
    }
    return Q;
}

/* out[A,i,n] += R_k Q_k(n) sum_{f,q} w N_a(q) n_i (rows of `free_only`-filtered nodes) */
static void resistance_apply(const hbo_problem* p, const double* v, double* out, int free_only) {
    if (!p->resistance)
        return;
    const int N = p->N, nk = neumann_entries(p);
    for (int k = 0; k < nk; ++k) {
        const double R = p->resistance[k];
        if (R == 0.0)
            continue;
        for (int n = 0; n < N; ++n) {
            const double RQ = R * entry_flux(p, k, v, n, free_only);
            for (int f = 0; f < p->nfac; ++f) {
                if (p->fbc[f] != k)
                    continue;
                const int* fac = p->fac + 3 * f;
                const double* nv = p->fnormal + 3 * f;
                const double w = p->farea[f] / 3.0;
                for (int q = 0; q < 3; ++q)
                    for (int a = 0; a < 3; ++a) {
                        if (free_only && p->dirichlet[fac[a]])
                            continue;
                        for (int i = 0; i < 3; ++i)
                            out[((size_t)fac[a] * 4 + i) * N + n] += w * tri_shape(q, a) * RQ * nv[i];
                    }
            }
        }
    }
}

int hbo_residual(const hbo_problem* p, const double* state, double* r) {
    const int N = p->N, nn = p->nn;
    const size_t tot = (size_t)nn * 4 * N;
    double* hu = malloc(sizeof(double) * (size_t)nn * 3 * N);
    double* s = calloc((size_t)nn * 3 * N, sizeof(double));
    memset(r, 0, sizeof(double) * tot);
    /* nodal H*u at every node (assembly.cpp:453-463) */
    for (int A = 0; A < nn; ++A)
        for (int i = 0; i < 3; ++i)
            apply_h(N, p->H, state + ((size_t)A * 4 + i) * N, hu + ((size_t)A * 3 + i) * N);
    int status = 0;
    for (int e = 0; e < p->ne && !status; ++e) {
        const int* cn = p->conn + 4 * e;
        const double* g = p->geom + 22 * (size_t)e;
        for (int n = 0; n < N && !status; ++n) {
            double u[4][3], pr[4], h4[4][3], rm[4][3] = {{0}}, rc[4] = {0}, sv[4][3] = {{0}};
            for (int a = 0; a < 4; ++a) {
                for (int i = 0; i < 3; ++i) {
                    u[a][i] = state[((size_t)cn[a] * 4 + i) * N + n];
                    h4[a][i] = hu[((size_t)cn[a] * 3 + i) * N + n];
                }
                pr[a] = state[((size_t)cn[a] * 4 + 3) * N + n];
            }
            if (element_residual_n(p, g, u, pr, h4, rm, rc, sv)) {
                status = -1;
                break;
            }
            /* scatter in element order (assembly.cpp:493-509) */
            for (int a = 0; a < 4; ++a) {
                for (int i = 0; i < 3; ++i) {
                    r[((size_t)cn[a] * 4 + i) * N + n] += rm[a][i];
                    s[((size_t)cn[a] * 3 + i) * N + n] += sv[a][i];
                }
                r[((size_t)cn[a] * 4 + 3) * N + n] += rc[a];
            }
        }
    }
    if (!status) {
        /* r_m -= H s (assembly.cpp:523-535) */
        double* hs = malloc(sizeof(double) * (size_t)N);
        for (int A = 0; A < nn; ++A)
            for (int i = 0; i < 3; ++i) {
                apply_h(N, p->H, s + ((size_t)A * 3 + i) * N, hs);
                for (int n = 0; n < N; ++n)
                    r[((size_t)A * 4 + i) * N + n] -= hs[n];
            }
        free(hs);
        boundary_terms(p, state, r);
        resistance_apply(p, state, r, 0);
        /* zero the constrained velocity rows (assembly.cpp:541-544) */
        for (int A = 0; A < nn; ++A)
            if (p->dirichlet[A])
                memset(r + (size_t)A * 4 * N, 0, sizeof(double) * 3 * (size_t)N);
    }
    free(hu);
    free(s);
    return status;
}

/* ---------------------------------------------------------------- tangent */

/* element_tangent_p (assembly.cpp:265-374) of one element at one time sample:
 * K[a][b], G[a][b][i], D[a][b][i], L[a][b] (assembly.hpp:101-110). */
static int element_tangent_n(const hbo_problem* p, const double* g, const double u[4][3],
                             double K[4][4], double G[4][4][3], double D[4][4][3],
                             double L[4][4]) {
    const double rho = p->rho, mu = p->mu, nu = mu / rho;
    const int pseudo = p->pseudo_dt > 0.0 && isfinite(p->pseudo_dt);
    const double pc = pseudo ? p->pseudo_c1 * rho / p->pseudo_dt : 0.0;
    const double V = GV(g), w = V / 4.0;
    double gg[4][4];
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            gg[a][b] = GN(g, a, 0) * GN(g, b, 0) + GN(g, a, 1) * GN(g, b, 1) +
                       GN(g, a, 2) * GN(g, b, 2);
            K[a][b] = mu * V * gg[a][b] + pc * (a == b ? V / 10.0 : V / 20.0);
            L[a][b] = 0.0;
            for (int i = 0; i < 3; ++i) {
                G[a][b][i] = -GN(g, a, i) * V / 4.0;
                D[a][b][i] = GN(g, b, i) * V / 4.0;
            }
        }
    double tau_mean = 0.0;
    if (p->tau_mode == 1) {
        double um[3] = {0, 0, 0};
        for (int a = 0; a < 4; ++a)
            for (int i = 0; i < 3; ++i)
                um[i] += 0.25 * u[a][i];
        if (tau_of(g, um, nu, &tau_mean))
            return -1;
    }
    for (int q = 0; q < 4; ++q) {
        double uq[3] = {0, 0, 0}, adv[4];
        for (int i = 0; i < 3; ++i)
            for (int a = 0; a < 4; ++a)
                uq[i] += tet_shape(q, a) * u[a][i];
        double tau = tau_mean;
        if (p->tau_mode == 0 && tau_of(g, uq, nu, &tau))
            return -1;
        for (int a = 0; a < 4; ++a)
            adv[a] = uq[0] * GN(g, a, 0) + uq[1] * GN(g, a, 1) + uq[2] * GN(g, a, 2);
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                K[a][b] += w * rho * (tet_shape(q, a) * adv[b] + adv[a] * tau * adv[b]);
                L[a][b] += w * gg[a][b] * tau / rho;
                for (int i = 0; i < 3; ++i) {
                    G[a][b][i] += w * adv[a] * tau * GN(g, b, i);
                    D[a][b][i] += w * GN(g, a, i) * tau * adv[b];
                }
            }
    }
    return 0;
}

int hbo_tangent(const hbo_problem* p, const int* row_ptr, const int* col_idx,
                const double* state, double* vals) {
    const int N = p->N;
    memset(vals, 0, sizeof(double) * (size_t)row_ptr[p->nn] * 8 * N);
    for (int e = 0; e < p->ne; ++e) {
        const int* cn = p->conn + 4 * e;
        const double* g = p->geom + 22 * (size_t)e;
        int blk[4][4];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b)
                blk[a][b] = hbo_find(row_ptr, col_idx, cn[a], cn[b]);
        for (int n = 0; n < N; ++n) {
            double u[4][3];
            for (int a = 0; a < 4; ++a)
                for (int i = 0; i < 3; ++i)
                    u[a][i] = state[((size_t)cn[a] * 4 + i) * N + n];
            double K[4][4], G[4][4][3], D[4][4][3], L[4][4];
            if (element_tangent_n(p, g, u, K, G, D, L))
                return -1;
            /* masked scatter (assembly.cpp:574-610) */
            for (int a = 0; a < 4; ++a) {
                const int afix = p->dirichlet[cn[a]] != 0;
                for (int b = 0; b < 4; ++b) {
                    const int bfix = p->dirichlet[cn[b]] != 0;
                    double* v = vals + (size_t)blk[a][b] * 8 * N + n;
                    if (!afix && !bfix)
                        v[0] += K[a][b];
                    for (int i = 0; i < 3; ++i) {
                        if (!afix)
                            v[(size_t)(1 + i) * N] += G[a][b][i];
                        if (!bfix)
                            v[(size_t)(4 + i) * N] += D[a][b][i];
                    }
                    v[(size_t)7 * N] += L[a][b];
                }
            }
        }
    }
    if (p->backflow_in_tangent) {
        /* frozen-coefficient backflow tangent (assembly.cpp:612-657) */
        for (int f = 0; f < p->nfac; ++f) {
            const int* fac = p->fac + 3 * f;
            const double* nv = p->fnormal + 3 * f;
            const double w = p->farea[f] / 3.0;
            for (int q = 0; q < 3; ++q)
                for (int n = 0; n < N; ++n) {
                    double uq[3] = {0, 0, 0};
                    for (int a = 0; a < 3; ++a)
                        for (int i = 0; i < 3; ++i)
                            uq[i] += tri_shape(q, a) * state[((size_t)fac[a] * 4 + i) * N + n];
                    const double un = uq[0] * nv[0] + uq[1] * nv[1] + uq[2] * nv[2];
                    if (!(un < 0.0))
                        continue;
                    for (int a = 0; a < 3; ++a) {
                        if (p->dirichlet[fac[a]])
                            continue;
                        for (int b = 0; b < 3; ++b) {
                            if (p->dirichlet[fac[b]])
                                continue;
                            const int k = hbo_find(row_ptr, col_idx, fac[a], fac[b]);
                            const double c = w * tri_shape(q, a) * tri_shape(q, b) * 0.5 *
                                             p->rho * p->beta;
                            vals[(size_t)k * 8 * N + n] -= c * un;
                        }
                    }
                }
        }
    }
    /* identity on constrained velocity diagonals (assembly.cpp:659-665) */
    for (int A = 0; A < p->nn; ++A)
        if (p->dirichlet[A]) {
            const int k = hbo_find(row_ptr, col_idx, A, A);
            for (int n = 0; n < N; ++n)
                vals[(size_t)k * 8 * N + n] = 1.0;
        }
    return 0;
}

void hbo_mass(const hbo_problem* p, const int* row_ptr, const int* col_idx, double* mass) {
    memset(mass, 0, sizeof(double) * (size_t)row_ptr[p->nn]);
    for (int e = 0; e < p->ne; ++e) {
        const int* cn = p->conn + 4 * e;
        const double V = GV(p->geom + 22 * (size_t)e);
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b)
                mass[hbo_find(row_ptr, col_idx, cn[a], cn[b])] +=
                    a == b ? p->rho * V / 10.0 : p->rho * V / 20.0;
    }
}

/* ---------------------------------------------------------------- operator */

void hbo_bsr_matvec(int nn, int N, const int* row_ptr, const int* col_idx, const double* vals,
                    const double* y, double* out) {
    for (int A = 0; A < nn; ++A) {
        double* o = out + (size_t)A * 4 * N;
        memset(o, 0, sizeof(double) * 4 * (size_t)N);
        for (int k = row_ptr[A]; k < row_ptr[A + 1]; ++k) {
            const double* v = vals + (size_t)k * 8 * N;
            const double* yb = y + (size_t)col_idx[k] * 4 * N;
            for (int n = 0; n < N; ++n) {
                const double yp = yb[3 * N + n];
                double op = v[7 * N + n] * yp;
                for (int i = 0; i < 3; ++i) {
                    o[i * N + n] += v[n] * yb[i * N + n] + v[(1 + i) * N + n] * yp;
                    op += v[(4 + i) * N + n] * yb[i * N + n];
                }
                o[3 * N + n] += op;
            }
        }
    }
}

void hbo_tangent_matvec(const hbo_problem* p, const int* row_ptr, const int* col_idx,
                        const double* vals, const double* mass, const double* y, double* out) {
    const int N = p->N;
    hbo_bsr_matvec(p->nn, N, row_ptr, col_idx, vals, y, out);
    double* t = malloc(sizeof(double) * 3 * (size_t)N);
    double* ht = malloc(sizeof(double) * (size_t)N);
    for (int A = 0; A < p->nn; ++A) {
        if (p->dirichlet[A])
            continue;
        memset(t, 0, sizeof(double) * 3 * (size_t)N);
        for (int k = row_ptr[A]; k < row_ptr[A + 1]; ++k) {
            const int B = col_idx[k];
            if (p->dirichlet[B])
                continue;
            for (int j = 0; j < 3 * N; ++j)
                t[j] += mass[k] * y[(size_t)B * 4 * N + j];
        }
        for (int i = 0; i < 3; ++i) {
            apply_h(N, p->H, t + i * N, ht);
            for (int n = 0; n < N; ++n)
                out[((size_t)A * 4 + i) * N + n] += ht[n];
        }
    }
    free(t);
    free(ht);
    resistance_apply(p, y, out, 1);
}

int hbo_jacobi(int nn, int N, const int* row_ptr, const int* col_idx, const double* vals,
               double* inv_diag) {
    int degenerate = 0;
    for (int A = 0; A < nn; ++A) {
        const int k = hbo_find(row_ptr, col_idx, A, A);
        for (int c = 0; c < 4; ++c)
            for (int n = 0; n < N; ++n) {
                const double d = vals[((size_t)k * 8 + (c < 3 ? 0 : 7)) * N + n];
                double* o = inv_diag + ((size_t)A * 4 + c) * N + n;
                if (fabs(d) < 1e-30) {
                    ++degenerate;
                    *o = 1.0;
                } else {
                    *o = 1.0 / d;
                }
            }
    }
    return degenerate;
}

/* ---------------------------------------------------------------- GMRES */

static double nrm2(long n, const double* v) {
    double s = 0.0;
    for (long i = 0; i < n; ++i)
        s += v[i] * v[i];
    return sqrt(s);
}

void hbo_gmres(hbo_apply_fn apply, void* user, long n, const double* rhs,
               const double* inv_diag, const hbo_krylov_cfg* cfg, double* x,
               hbo_krylov_result* res, double* history) {
    /* split Jacobi scaling S = diag(sqrt|inv_diag|), (S A S) w = S b, x = S w;
     * restarted, modified Gram-Schmidt, Givens (linalg.cpp:167-293). */
    const int m = cfg->restart > 1 ? cfg->restart : 1;
    res->iterations = 0;
    res->relative_residual = 1.0;
    res->status = 0;
    res->history_len = 0;
    double* sc = malloc(sizeof(double) * (size_t)n);
    double* b = malloc(sizeof(double) * (size_t)n);
    for (long i = 0; i < n; ++i) {
        x[i] = 0.0;
        sc[i] = sqrt(fabs(inv_diag[i]));
        b[i] = sc[i] * rhs[i];
    }
    const double bnorm = nrm2(n, b);
    if (bnorm == 0.0) {
        res->relative_residual = 0.0;
        free(sc);
        free(b);
        return;
    }
    double* V = malloc(sizeof(double) * (size_t)n * (size_t)(m + 1));
    double* Hs = malloc(sizeof(double) * (size_t)(m + 1) * (size_t)m);
    double* cs = malloc(sizeof(double) * (size_t)m);
    double* sn = malloc(sizeof(double) * (size_t)m);
    double* gv = malloc(sizeof(double) * (size_t)(m + 1));
    double* yv = malloc(sizeof(double) * (size_t)m);
    double* r = malloc(sizeof(double) * (size_t)n);
    double* w = malloc(sizeof(double) * (size_t)n);
    double* z = malloc(sizeof(double) * (size_t)n);
    memcpy(r, b, sizeof(double) * (size_t)n);
    double rnorm = bnorm;
    history[res->history_len++] = 1.0;
#define HH(i, j) Hs[(size_t)(j) * (size_t)(m + 1) + (size_t)(i)]
    while (res->iterations < cfg->max_iters) {
        const double cycle_start = rnorm;
        memset(Hs, 0, sizeof(double) * (size_t)(m + 1) * (size_t)m);
        memset(gv, 0, sizeof(double) * (size_t)(m + 1));
        gv[0] = rnorm;
        for (long i = 0; i < n; ++i)
            V[i] = r[i] / rnorm;
        int j = 0;
        for (; j < m && res->iterations < cfg->max_iters; ++j) {
            const double* vj = V + (size_t)j * (size_t)n;
            for (long i = 0; i < n; ++i)
                z[i] = sc[i] * vj[i];
            apply(user, z, w);
            for (long i = 0; i < n; ++i)
                w[i] *= sc[i];
            for (int i = 0; i <= j; ++i) {
                const double* vi = V + (size_t)i * (size_t)n;
                double h = 0.0;
                for (long k = 0; k < n; ++k)
                    h += w[k] * vi[k];
                HH(i, j) = h;
                for (long k = 0; k < n; ++k)
                    w[k] -= h * vi[k];
            }
            const double hj1 = nrm2(n, w);
            HH(j + 1, j) = hj1;
            if (hj1 > 0.0) {
                double* vn = V + (size_t)(j + 1) * (size_t)n;
                for (long k = 0; k < n; ++k)
                    vn[k] = w[k] / hj1;
            }
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * HH(i, j) + sn[i] * HH(i + 1, j);
                HH(i + 1, j) = -sn[i] * HH(i, j) + cs[i] * HH(i + 1, j);
                HH(i, j) = t;
            }
            const double den = hypot(HH(j, j), HH(j + 1, j));
            cs[j] = den == 0.0 ? 1.0 : HH(j, j) / den;
            sn[j] = den == 0.0 ? 0.0 : HH(j + 1, j) / den;
            HH(j, j) = den;
            HH(j + 1, j) = 0.0;
            gv[j + 1] = -sn[j] * gv[j];
            gv[j] = cs[j] * gv[j];
            res->iterations += 1;
            const double est = fabs(gv[j + 1]);
            history[res->history_len++] = est / bnorm;
            if (est / bnorm <= cfg->tolerance || hj1 == 0.0) {
                ++j;
                break;
            }
        }
        while (j > 0 && HH(j - 1, j - 1) == 0.0)
            --j;
        for (int i = j - 1; i >= 0; --i) {
            double s = gv[i];
            for (int k = i + 1; k < j; ++k)
                s -= HH(i, k) * yv[k];
            yv[i] = s / HH(i, i);
        }
        for (int i = 0; i < j; ++i) {
            const double* vi = V + (size_t)i * (size_t)n;
            for (long k = 0; k < n; ++k)
                x[k] += sc[k] * vi[k] * yv[i];
        }
        apply(user, x, w);
        for (long k = 0; k < n; ++k)
            r[k] = sc[k] * (rhs[k] - w[k]);
        rnorm = nrm2(n, r);
        res->relative_residual = rnorm / bnorm;
        if (res->relative_residual <= cfg->tolerance) {
            res->status = 0;
            goto done;
        }
        if (rnorm >= cycle_start) {
            res->status = 2;
            goto done;
        }
    }
    res->status = 1;
done:
#undef HH
    free(sc);
    free(b);
    free(V);
    free(Hs);
    free(cs);
    free(sn);
    free(gv);
    free(yv);
    free(r);
    free(w);
    free(z);
}

typedef struct {
    const hbo_problem* p;
    const int* row_ptr;
    const int* col_idx;
    const double* vals;
    const double* mass;
} tangent_user;

static void tangent_apply(void* u, const double* y, double* out) {
    const tangent_user* t = (const tangent_user*)u;
    hbo_tangent_matvec(t->p, t->row_ptr, t->col_idx, t->vals, t->mass, y, out);
}

void hbo_gmres_tangent(const hbo_problem* p, const int* row_ptr, const int* col_idx,
                       const double* vals, const double* mass, const double* rhs,
                       const double* inv_diag, const hbo_krylov_cfg* cfg, double* x,
                       hbo_krylov_result* res, double* history) {
    tangent_user u = {p, row_ptr, col_idx, vals, mass};
    hbo_gmres(tangent_apply, &u, (long)p->nn * 4 * p->N, rhs, inv_diag, cfg, x, res, history);
}

/* ---------------------------------------------------------------- time solver */

/* time_solver.cpp:34-43: (omega_hat^2 + u.xi.u + 3 nu^2 xi:xi)^(-1/2), full 3x3 xi */
static double tau_hat_of(const double* g, const double u[3], double nu, double omega_hat) {
    double conv = 0.0, xx = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double x = g[13 + 3 * i + j];
            conv += u[i] * x * u[j];
            xx += x * x;
        }
    return 1.0 / sqrt(omega_hat * omega_hat + conv + 3.0 * nu * nu * xx);
}

void hbo_time_residual(const hbo_problem* p, const double* u, const double* udot, const double* pres,
                       double omega_hat, double* r) {
    const double rho = p->rho, mu = p->mu, nu = mu / rho;
    memset(r, 0, sizeof(double) * (size_t)p->nn * 4);
    for (int e = 0; e < p->ne; ++e) {
        const int* cn = p->conn + 4 * e;
        const double* g = p->geom + 22 * (size_t)e;
        const double w = g[12] / 4.0;
        double gu[3][3] = {{0}}, gp[3] = {0};
        for (int a = 0; a < 4; ++a)
            for (int i = 0; i < 3; ++i) {
                for (int j = 0; j < 3; ++j)
                    gu[i][j] += GN(g, a, j) * u[3 * (size_t)cn[a] + i];
                gp[i] += GN(g, a, i) * pres[cn[a]];
            }
        const double divu = gu[0][0] + gu[1][1] + gu[2][2];
        for (int q = 0; q < 4; ++q) {
            double uq[3] = {0, 0, 0}, aq[3] = {0, 0, 0}, pq = 0.0;
            for (int a = 0; a < 4; ++a) {
                const double sa = tet_shape(q, a);
                for (int i = 0; i < 3; ++i) {
                    uq[i] += sa * u[3 * (size_t)cn[a] + i];
                    aq[i] += sa * udot[3 * (size_t)cn[a] + i];
                }
                pq += sa * pres[cn[a]];
            }
            const double th = tau_hat_of(g, uq, nu, omega_hat);
            double lq[3];
            for (int i = 0; i < 3; ++i) {
                double cv = 0.0;
                for (int j = 0; j < 3; ++j)
                    cv += uq[j] * gu[i][j];
                lq[i] = rho * aq[i] + rho * cv + gp[i];
            }
            for (int a = 0; a < 4; ++a) {
                const double sa = tet_shape(q, a);
                double adv = 0.0;
                for (int j = 0; j < 3; ++j)
                    adv += uq[j] * GN(g, a, j);
                for (int i = 0; i < 3; ++i) {
                    double cv = 0.0, visc = 0.0;
                    for (int j = 0; j < 3; ++j) {
                        cv += uq[j] * gu[i][j];
                        visc += GN(g, a, j) * gu[i][j];
                    }
                    r[4 * (size_t)cn[a] + i] +=
                        w * (rho * sa * (aq[i] + cv) - GN(g, a, i) * pq + mu * visc + adv * th * lq[i]);
                }
                double pspg = 0.0;
                for (int i = 0; i < 3; ++i)
                    pspg += GN(g, a, i) * th * lq[i];
                r[4 * (size_t)cn[a] + 3] += w * (sa * divu + pspg / rho);
            }
        }
    }
    /* Neumann traction (steady h[0]) and backflow (time_solver.cpp:130-160) */
    for (int f = 0; f < p->nfac; ++f) {
        const int* fac = p->fac + 3 * f;
        const double* nv = p->fnormal + 3 * f;
        const double h = p->h[(size_t)p->fbc[f] * p->N];
        const double w = p->farea[f] / 3.0;
        for (int q = 0; q < 3; ++q) {
            double uq[3] = {0, 0, 0};
            for (int a = 0; a < 3; ++a)
                for (int i = 0; i < 3; ++i)
                    uq[i] += tri_shape(q, a) * u[3 * (size_t)fac[a] + i];
            const double un = uq[0] * nv[0] + uq[1] * nv[1] + uq[2] * nv[2];
            const double neg = un < 0.0 ? un : 0.0;
            for (int a = 0; a < 3; ++a)
                for (int i = 0; i < 3; ++i)
                    r[4 * (size_t)fac[a] + i] +=
                        w * tri_shape(q, a) * (-h * nv[i] - 0.5 * rho * p->beta * neg * uq[i]);
        }
    }
    for (int A = 0; A < p->nn; ++A)
        if (p->dirichlet[A])
            for (int i = 0; i < 3; ++i)
                r[4 * (size_t)A + i] = 0.0;
}

void hbo_time_tangent(const hbo_problem* p, const int* row_ptr, const int* col_idx, const double* u,
                      double omega_hat, double am, double fg, double* vals) {
    const double rho = p->rho, mu = p->mu, nu = mu / rho;
    memset(vals, 0, sizeof(double) * (size_t)row_ptr[p->nn] * 8);
    for (int e = 0; e < p->ne; ++e) {
        const int* cn = p->conn + 4 * e;
        const double* g = p->geom + 22 * (size_t)e;
        const double V = g[12], w = V / 4.0;
        double K[16] = {0}, G[16][3] = {{0}}, D[16][3] = {{0}}, L[16] = {0};
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                double gg = 0.0;
                for (int j = 0; j < 3; ++j)
                    gg += GN(g, a, j) * GN(g, b, j);
                const double m = a == b ? V / 10.0 : V / 20.0; /* element_mass(g, 1), assembly.cpp:58-66 */
                K[a * 4 + b] += am * rho * m + fg * mu * V * gg;
                L[a * 4 + b] = 0.0;
                for (int i = 0; i < 3; ++i) {
                    G[a * 4 + b][i] += -GN(g, a, i) * V / 4.0;
                    D[a * 4 + b][i] += fg * GN(g, b, i) * V / 4.0;
                }
            }
        for (int q = 0; q < 4; ++q) {
            double uq[3] = {0, 0, 0};
            for (int a = 0; a < 4; ++a)
                for (int i = 0; i < 3; ++i)
                    uq[i] += tet_shape(q, a) * u[3 * (size_t)cn[a] + i];
            const double th = tau_hat_of(g, uq, nu, omega_hat);
            double adv[4];
            for (int a = 0; a < 4; ++a) {
                adv[a] = 0.0;
                for (int j = 0; j < 3; ++j)
                    adv[a] += uq[j] * GN(g, a, j);
            }
            for (int a = 0; a < 4; ++a) {
                const double sa = tet_shape(q, a);
                for (int b = 0; b < 4; ++b) {
                    const double sb = tet_shape(q, b);
                    K[a * 4 + b] += w * (fg * rho * (sa * adv[b] + adv[a] * th * adv[b]) + am * rho * adv[a] * th * sb);
                    double gg = 0.0;
                    for (int j = 0; j < 3; ++j)
                        gg += GN(g, a, j) * GN(g, b, j);
                    L[a * 4 + b] += w * gg * th / rho;
                    for (int i = 0; i < 3; ++i) {
                        G[a * 4 + b][i] += w * adv[a] * th * GN(g, b, i);
                        D[a * 4 + b][i] += w * GN(g, a, i) * th * (am * sb + fg * adv[b]);
                    }
                }
            }
        }
        for (int a = 0; a < 4; ++a) {
            const int A = cn[a];
            const int afix = p->dirichlet[A] != 0;
            for (int b = 0; b < 4; ++b) {
                const int B = cn[b];
                const int bfix = p->dirichlet[B] != 0;
                double* v = vals + 8 * (size_t)hbo_find(row_ptr, col_idx, A, B);
                if (!afix && !bfix)
                    v[0] += K[a * 4 + b];
                for (int i = 0; i < 3; ++i) {
                    if (!afix)
                        v[1 + i] += G[a * 4 + b][i];
                    if (!bfix)
                        v[4 + i] += D[a * 4 + b][i];
                }
                v[7] += L[a * 4 + b];
            }
        }
    }
    for (int A = 0; A < p->nn; ++A)
        if (p->dirichlet[A])
            vals[8 * (size_t)hbo_find(row_ptr, col_idx, A, A)] = 1.0;
}

/* ---------------------------------------------------------------- row subsets
 *
 * The residual rows and P block rows of a given node list, computed with the
 * same per-entry summation order as hbo_residual / hbo_tangent (element order,
 * then facet order), so each returned entry is bit-identical to the full
 * assembly's.  They exist so that parity can be checked on full-size meshes
 * (millions of elements, P.vals beyond 2^31 doubles) in seconds. */

/* Elements incident to each listed row, ascending: CSR (ptr[nrows+1], elem). */
static int incident_elements(const hbo_problem* p, int nrows, const int* rows, int** ptr_out,
                             int** elem_out) {
    int* slot = malloc(sizeof(int) * (size_t)p->nn);
    int* ptr = calloc((size_t)nrows + 1, sizeof(int));
    if (!slot || !ptr) {
        free(slot);
        free(ptr);
        return -1;
    }
    for (int A = 0; A < p->nn; ++A)
        slot[A] = -1;
    for (int k = 0; k < nrows; ++k) {
        if (rows[k] < 0 || rows[k] >= p->nn || slot[rows[k]] >= 0) {
            free(slot);
            free(ptr);
            return -2; /* out of range or repeated */
        }
        slot[rows[k]] = k;
    }
    for (int e = 0; e < p->ne; ++e)
        for (int a = 0; a < 4; ++a) {
            const int k = slot[p->conn[4 * e + a]];
            if (k >= 0)
                ptr[k + 1] += 1;
        }
    for (int k = 0; k < nrows; ++k)
        ptr[k + 1] += ptr[k];
    int* elem = malloc(sizeof(int) * (size_t)(ptr[nrows] > 0 ? ptr[nrows] : 1));
    int* fill = malloc(sizeof(int) * (size_t)(nrows > 0 ? nrows : 1));
    for (int k = 0; k < nrows; ++k)
        fill[k] = ptr[k];
    for (int e = 0; e < p->ne; ++e)
        for (int a = 0; a < 4; ++a) {
            const int k = slot[p->conn[4 * e + a]];
            if (k >= 0)
                elem[fill[k]++] = e;
        }
    free(fill);
    free(slot);
    *ptr_out = ptr;
    *elem_out = elem;
    return 0;
}

static int local_index(const int* cn, int A) {
    for (int a = 0; a < 4; ++a)
        if (cn[a] == A)
            return a;
    return -1;
}

int hbo_residual_rows(const hbo_problem* p, const double* state, int nrows, const int* rows,
                      double* r) {
    const int N = p->N;
    if (N > 64)
        return -3;
    int *ptr, *elem;
    const int st = incident_elements(p, nrows, rows, &ptr, &elem);
    if (st)
        return st;
    double* s = malloc(sizeof(double) * 3 * (size_t)N);
    double* hs = malloc(sizeof(double) * (size_t)N);
    int status = 0;
    for (int k = 0; k < nrows && !status; ++k) {
        const int A = rows[k];
        double* rA = r + (size_t)k * 4 * N;
        memset(rA, 0, sizeof(double) * 4 * (size_t)N);
        memset(s, 0, sizeof(double) * 3 * (size_t)N);
        for (int t = ptr[k]; t < ptr[k + 1] && !status; ++t) {
            const int e = elem[t];
            const int* cn = p->conn + 4 * e;
            const double* g = p->geom + 22 * (size_t)e;
            const int la = local_index(cn, A);
            /* nodal H*u of the element's nodes (assembly.cpp:453-463) */
            double hu4[4][3][64];
            for (int a = 0; a < 4; ++a)
                for (int i = 0; i < 3; ++i)
                    apply_h(N, p->H, state + ((size_t)cn[a] * 4 + i) * N, hu4[a][i]);
            for (int n = 0; n < N; ++n) {
                double u[4][3], pr[4], h4[4][3], rm[4][3] = {{0}}, rc[4] = {0}, sv[4][3] = {{0}};
                for (int a = 0; a < 4; ++a) {
                    for (int i = 0; i < 3; ++i) {
                        u[a][i] = state[((size_t)cn[a] * 4 + i) * N + n];
                        h4[a][i] = hu4[a][i][n];
                    }
                    pr[a] = state[((size_t)cn[a] * 4 + 3) * N + n];
                }
                if (element_residual_n(p, g, u, pr, h4, rm, rc, sv)) {
                    status = -1;
                    break;
                }
                for (int i = 0; i < 3; ++i) {
                    rA[(size_t)i * N + n] += rm[la][i];
                    s[(size_t)i * N + n] += sv[la][i];
                }
                rA[(size_t)3 * N + n] += rc[la];
            }
        }
        if (status)
            break;
        /* r_m -= H s (assembly.cpp:523-535) */
        for (int i = 0; i < 3; ++i) {
            apply_h(N, p->H, s + (size_t)i * N, hs);
            for (int n = 0; n < N; ++n)
                rA[(size_t)i * N + n] -= hs[n];
        }
        /* Neumann traction + backflow of the facets touching A (assembly.cpp:376-413) */
        for (int f = 0; f < p->nfac; ++f) {
            const int* fac = p->fac + 3 * f;
            int la = -1;
            for (int a = 0; a < 3; ++a)
                if (fac[a] == A)
                    la = a;
            if (la < 0)
                continue;
            const double* nv = p->fnormal + 3 * f;
            const double* h = p->h + (size_t)p->fbc[f] * N;
            const double w = p->farea[f] / 3.0;
            for (int q = 0; q < 3; ++q)
                for (int n = 0; n < N; ++n) {
                    double uq[3] = {0, 0, 0};
                    for (int a = 0; a < 3; ++a)
                        for (int i = 0; i < 3; ++i)
                            uq[i] += tri_shape(q, a) * state[((size_t)fac[a] * 4 + i) * N + n];
                    const double un = uq[0] * nv[0] + uq[1] * nv[1] + uq[2] * nv[2];
                    const double neg = un < 0.0 ? un : 0.0;
                    for (int i = 0; i < 3; ++i)
                        rA[(size_t)i * N + n] += w * tri_shape(q, la) *
                                                 (-h[n] * nv[i] - 0.5 * p->rho * p->beta * neg * uq[i]);
                }
        }
        /* resistance outlets (see hbgls_oracle.h) */
        if (p->resistance) {
            const int nk = neumann_entries(p);
            for (int kk = 0; kk < nk; ++kk) {
                const double R = p->resistance[kk];
                if (R == 0.0)
                    continue;
                for (int n = 0; n < N; ++n) {
                    const double RQ = R * entry_flux(p, kk, state, n, 0);
                    for (int f = 0; f < p->nfac; ++f) {
                        if (p->fbc[f] != kk)
                            continue;
                        const int* fac = p->fac + 3 * f;
                        const double* nv = p->fnormal + 3 * f;
                        const double w = p->farea[f] / 3.0;
                        for (int q = 0; q < 3; ++q)
                            for (int a = 0; a < 3; ++a) {
                                if (fac[a] != A)
                                    continue;
                                for (int i = 0; i < 3; ++i)
                                    rA[(size_t)i * N + n] += w * tri_shape(q, a) * RQ * nv[i];
                            }
                    }
                }
            }
        }
        if (p->dirichlet[A])
            memset(rA, 0, sizeof(double) * 3 * (size_t)N);
    }
    free(s);
    free(hs);
    free(ptr);
    free(elem);
    return status;
}

int hbo_tangent_rows(const hbo_problem* p, const int* row_ptr, const int* col_idx,
                     const double* state, int nrows, const int* rows, double* vals) {
    const int N = p->N;
    int *ptr, *elem;
    const int st = incident_elements(p, nrows, rows, &ptr, &elem);
    if (st)
        return st;
    size_t off = 0;
    int status = 0;
    for (int k = 0; k < nrows && !status; ++k) {
        const int A = rows[k];
        const int r0 = row_ptr[A], nb = row_ptr[A + 1] - r0;
        double* vA = vals + off;
        off += (size_t)nb * 8 * N;
        memset(vA, 0, sizeof(double) * (size_t)nb * 8 * N);
        const int afix = p->dirichlet[A] != 0;
        for (int t = ptr[k]; t < ptr[k + 1] && !status; ++t) {
            const int e = elem[t];
            const int* cn = p->conn + 4 * e;
            const double* g = p->geom + 22 * (size_t)e;
            const int la = local_index(cn, A);
            int blk[4];
            for (int b = 0; b < 4; ++b)
                blk[b] = hbo_find(row_ptr, col_idx, A, cn[b]) - r0;
            for (int n = 0; n < N; ++n) {
                double u[4][3];
                for (int a = 0; a < 4; ++a)
                    for (int i = 0; i < 3; ++i)
                        u[a][i] = state[((size_t)cn[a] * 4 + i) * N + n];
                double K[4][4], G[4][4][3], D[4][4][3], L[4][4];
                if (element_tangent_n(p, g, u, K, G, D, L)) {
                    status = -1;
                    break;
                }
                for (int b = 0; b < 4; ++b) {
                    const int bfix = p->dirichlet[cn[b]] != 0;
                    double* v = vA + (size_t)blk[b] * 8 * N + n;
                    if (!afix && !bfix)
                        v[0] += K[la][b];
                    for (int i = 0; i < 3; ++i) {
                        if (!afix)
                            v[(size_t)(1 + i) * N] += G[la][b][i];
                        if (!bfix)
                            v[(size_t)(4 + i) * N] += D[la][b][i];
                    }
                    v[(size_t)7 * N] += L[la][b];
                }
            }
        }
        if (status)
            break;
        if (p->backflow_in_tangent && !afix) {
            /* frozen-coefficient backflow tangent (assembly.cpp:612-657), row A */
            for (int f = 0; f < p->nfac; ++f) {
                const int* fac = p->fac + 3 * f;
                int la = -1;
                for (int a = 0; a < 3; ++a)
                    if (fac[a] == A)
                        la = a;
                if (la < 0)
                    continue;
                const double* nv = p->fnormal + 3 * f;
                const double w = p->farea[f] / 3.0;
                for (int q = 0; q < 3; ++q)
                    for (int n = 0; n < N; ++n) {
                        double uq[3] = {0, 0, 0};
                        for (int a = 0; a < 3; ++a)
                            for (int i = 0; i < 3; ++i)
                                uq[i] += tri_shape(q, a) * state[((size_t)fac[a] * 4 + i) * N + n];
                        const double un = uq[0] * nv[0] + uq[1] * nv[1] + uq[2] * nv[2];
                        if (!(un < 0.0))
                            continue;
                        for (int b = 0; b < 3; ++b) {
                            if (p->dirichlet[fac[b]])
                                continue;
                            const int kb = hbo_find(row_ptr, col_idx, A, fac[b]) - r0;
                            const double c = w * tri_shape(q, la) * tri_shape(q, b) * 0.5 * p->rho *
                                             p->beta;
                            vA[(size_t)kb * 8 * N + n] -= c * un;
                        }
                    }
            }
        }
        if (afix) {
            /* identity on constrained velocity diagonals (assembly.cpp:659-665) */
            const int kd = hbo_find(row_ptr, col_idx, A, A) - r0;
            for (int n = 0; n < N; ++n)
                vA[(size_t)kd * 8 * N + n] = 1.0;
        }
    }
    free(ptr);
    free(elem);
    return status;
}

int hbo_tangent_matvec_rows(const hbo_problem* p, const int* row_ptr, const int* col_idx,
                            const double* row_vals, const double* mass, const double* y, int nrows,
                            const int* rows, double* out) {
    const int N = p->N;
    double* t = malloc(sizeof(double) * 3 * (size_t)N);
    double* ht = malloc(sizeof(double) * (size_t)N);
    size_t off = 0;
    for (int r = 0; r < nrows; ++r) {
        const int A = rows[r];
        if (A < 0 || A >= p->nn) {
            free(t);
            free(ht);
            return -2;
        }
        double* o = out + (size_t)r * 4 * N;
        memset(o, 0, sizeof(double) * 4 * (size_t)N);
        /* BlockSparseMatrix::matvec row A (linalg.cpp:41-76) */
        for (int k = row_ptr[A]; k < row_ptr[A + 1]; ++k) {
            const double* v = row_vals + off + (size_t)(k - row_ptr[A]) * 8 * N;
            const double* yb = y + (size_t)col_idx[k] * 4 * N;
            for (int n = 0; n < N; ++n) {
                const double yp = yb[3 * N + n];
                double op = v[7 * N + n] * yp;
                for (int i = 0; i < 3; ++i) {
                    o[i * N + n] += v[n] * yb[i * N + n] + v[(1 + i) * N + n] * yp;
                    op += v[(4 + i) * N + n] * yb[i * N + n];
                }
                o[3 * N + n] += op;
            }
        }
        off += (size_t)(row_ptr[A + 1] - row_ptr[A]) * 8 * N;
        if (p->dirichlet[A])
            continue;
        /* H (x) mass part (linalg.cpp:84-127) */
        memset(t, 0, sizeof(double) * 3 * (size_t)N);
        for (int k = row_ptr[A]; k < row_ptr[A + 1]; ++k) {
            const int B = col_idx[k];
            if (p->dirichlet[B])
                continue;
            for (int j = 0; j < 3 * N; ++j)
                t[j] += mass[k] * y[(size_t)B * 4 * N + j];
        }
        for (int i = 0; i < 3; ++i) {
            apply_h(N, p->H, t + i * N, ht);
            for (int n = 0; n < N; ++n)
                o[(size_t)i * N + n] += ht[n];
        }
        /* resistance outlets, free rows and columns (see hbgls_oracle.h) */
        if (p->resistance) {
            const int nk = neumann_entries(p);
            for (int kk = 0; kk < nk; ++kk) {
                const double R = p->resistance[kk];
                if (R == 0.0)
                    continue;
                for (int n = 0; n < N; ++n) {
                    const double RQ = R * entry_flux(p, kk, y, n, 1);
                    for (int f = 0; f < p->nfac; ++f) {
                        if (p->fbc[f] != kk)
                            continue;
                        const int* fac = p->fac + 3 * f;
                        const double* nv = p->fnormal + 3 * f;
                        const double w = p->farea[f] / 3.0;
                        for (int q = 0; q < 3; ++q)
                            for (int a = 0; a < 3; ++a) {
                                if (fac[a] != A)
                                    continue;
                                for (int i = 0; i < 3; ++i)
                                    o[(size_t)i * N + n] += w * tri_shape(q, a) * RQ * nv[i];
                            }
                    }
                }
            }
        }
    }
    free(t);
    free(ht);
    return 0;
}
