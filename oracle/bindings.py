"""ctypes bindings for the two CPU oracles — TEST INFRASTRUCTURE ONLY.

* `Ref*`   -> oracle/_ref/libhbref.so, the reference compiled from
             /root/reference/proj (oracle/Makefile, oracle/ref_capi.cpp).
* `Restated` -> oracle/_ref/libhboracle.so, the plain-C restatement
             (oracle/hbgls_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
legs may import this module.  Nothing in paper_2411_14315_b200/ does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libhbref.so")
ORACLE_SO = os.path.join(HERE, "_ref", "libhboracle.so")

_vp = C.c_void_p
_i = C.c_int
_d = C.c_double


def _ptr(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


# ------------------------------------------------------------------ reference

class _RefLib:
    _inst = None

    @classmethod
    def get(cls):
        if cls._inst is None:
            cls._inst = cls()
        return cls._inst

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise OracleError(f"{REF_SO} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(REF_SO)
        self.L = L
        s = lambda n, r, a: _sig(L, n, r, a)  # noqa: E731
        self.last_error = s("hbref_last_error", C.c_char_p, [])
        self.mesh_create = s("hbref_mesh_create", _vp, [_i, _vp, _i, _vp, _i, C.c_char_p, _vp, _vp, _vp])
        self.mesh_tube = s("hbref_mesh_tube", _vp, [_d, _d, _d])
        self.mesh_bif = s("hbref_mesh_bifurcation", _vp, [_d, _d, _d, _d, _d])
        self.mesh_destroy = s("hbref_mesh_destroy", None, [_vp])
        self.mesh_sizes = s("hbref_mesh_sizes", _i, [_vp, _vp, _vp, _vp, _vp])
        self.mesh_export = s("hbref_mesh_export", _i, [_vp] + [_vp] * 8)
        self.patch_name = s("hbref_patch_name", _i, [_vp, _i, C.c_char_p, _i])
        self.geometry = s("hbref_geometry", _i, [_vp, _vp])
        self.char_len = s("hbref_characteristic_length", _d, [_vp])
        self.pattern = s("hbref_pattern", _i, [_vp, _vp, _vp, _vp])
        self.h_dense = s("hbref_h_dense", _i, [_i, _d, _vp])
        self.oracle_h_dense = s("hbref_oracle_h_dense", _i, [_i, _d, _vp])
        self.apply_h = s("hbref_apply_h", _i, [_i, _d, _vp, _vp, _i])
        self.ctx_create = s("hbref_ctx_create", _vp, [_vp, _i, _d, _d, _d])
        self.ctx_destroy = s("hbref_ctx_destroy", None, [_vp])
        self.set_bcs = s("hbref_ctx_set_bcs", _i, [_vp, _vp, _i, _vp, _vp, _d])
        self.set_cfg = s("hbref_ctx_set_cfg", _i, [_vp, _i, _d, _d, _i])
        self.residual = s("hbref_residual", _i, [_vp, _vp, _i, _vp])
        self.oracle_residual = s("hbref_oracle_residual", _i, [_vp, _vp, _vp])
        self.frozen_residual = s("hbref_frozen_residual", _i, [_vp, _vp, _vp, _vp])
        self.tangent = s("hbref_tangent", _i, [_vp, _vp, _vp])
        self.pvals_size = s("hbref_pvals_size", C.c_longlong, [_vp])
        self.set_pvals = s("hbref_set_pvals", _i, [_vp, _vp])
        self.mass = s("hbref_mass", _i, [_vp, _vp])
        self.matvec = s("hbref_matvec", _i, [_vp, _vp, _vp, _i])
        self.bsr_matvec = s("hbref_bsr_matvec", _i, [_vp, _vp, _vp, _i])
        self.jacobi = s("hbref_jacobi", _i, [_vp, _vp, _vp])
        self.gmres = s("hbref_gmres", _i, [_vp, _vp, _vp, _i, _i, _d, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp])
        self.install_dirichlet = s("hbref_install_dirichlet", _i, [_vp, _vp])
        self.initial_pressure = s("hbref_initial_pressure", _d, [_vp])
        self.suggest_dt = s("hbref_suggest_pseudo_dt", _d, [_vp])
        self.dense_tangent = s("hbref_dense_tangent", _i, [_vp, _vp, _vp])
        self.solve = s("hbref_solve", _i, [_vp, _d, _d, _i, _i, _i, _d, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp])
        self.solve_time = s("hbref_solve_time", _i, [_vp, _d, _i, _i, _d, _d, _i, _i, _i, _d, _i, _i, _vp, _vp,
                                                     _vp, _vp, _vp])

    def check(self, st):
        if st != 0:
            raise OracleError(f"reference status {st}: {self.last_error().decode()}")


class RefMesh:
    """A reference `Mesh` (finalized by the reference's own Mesh::finalize)."""

    def __init__(self, handle):
        self.R = _RefLib.get()
        if not handle:
            raise OracleError(self.R.last_error().decode())
        self.h = handle

    @classmethod
    def from_mesh(cls, mesh):
        R = _RefLib.get()
        xyz = _f64(mesh.xyz)
        conn = np.ascontiguousarray(mesh.conn, dtype=np.int32)
        names = "\n".join(p.name for p in mesh.patches).encode()
        kinds = np.array([p.kind for p in mesh.patches], np.int32)
        nf = np.array([len(p.facets) for p in mesh.patches], np.int32)
        fac = np.ascontiguousarray(np.concatenate([p.facets for p in mesh.patches]), np.int32)
        return cls(R.mesh_create(mesh.num_nodes, _ptr(xyz), mesh.num_elements, _ptr(conn),
                                 len(mesh.patches), names, _ptr(kinds), _ptr(nf), _ptr(fac)))

    @classmethod
    def tube(cls, radius, length, h):
        return cls(_RefLib.get().mesh_tube(radius, length, h))

    @classmethod
    def bifurcation(cls, width, depth, inlet_length, branch_length, h):
        return cls(_RefLib.get().mesh_bif(width, depth, inlet_length, branch_length, h))

    def __del__(self):
        if getattr(self, "h", None):
            self.R.mesh_destroy(self.h)
            self.h = None

    def sizes(self):
        v = [C.c_int() for _ in range(4)]
        self.R.mesh_sizes(self.h, *[C.byref(x) for x in v])
        return [x.value for x in v]

    def to_mesh(self):
        """Export as a paper_2411_14315_b200.mesh.Mesh (already finalized)."""
        from paper_2411_14315_b200.mesh import Mesh, Patch

        nn, ne, npch, tf = self.sizes()
        xyz = np.empty((nn, 3))
        conn = np.empty((ne, 4), np.int32)
        kinds = np.empty(npch, np.int32)
        nf = np.empty(npch, np.int32)
        fac = np.empty((tf, 3), np.int32)
        nrm = np.empty((tf, 3))
        area = np.empty(tf)
        dm = np.empty(nn, np.uint8)
        self.R.check(self.R.mesh_export(self.h, _ptr(xyz), _ptr(conn), _ptr(kinds), _ptr(nf),
                                        _ptr(fac), _ptr(nrm), _ptr(area), _ptr(dm)))
        patches, off = [], 0
        for p in range(npch):
            buf = C.create_string_buffer(256)
            self.R.patch_name(self.h, p, buf, 256)
            k = int(nf[p])
            patches.append(Patch(buf.value.decode(), int(kinds[p]), fac[off:off + k].copy(),
                                 nrm[off:off + k].copy(), area[off:off + k].copy()))
            off += k
        return Mesh(xyz, conn, patches, dm)

    def geometry(self):
        ne = self.sizes()[1]
        g = np.empty((ne, 22))
        self.R.check(self.R.geometry(self.h, _ptr(g)))
        return g

    def characteristic_length(self):
        return self.R.char_len(self.h)

    def pattern(self):
        nn = self.sizes()[0]
        nnz = C.c_int()
        rp = np.empty(nn + 1, np.int32)
        self.R.check(self.R.pattern(self.h, _ptr(rp), None, C.byref(nnz)))
        ci = np.empty(nnz.value, np.int32)
        self.R.check(self.R.pattern(self.h, None, _ptr(ci), C.byref(nnz)))
        return rp, ci


def ref_h_dense(modes, period=1.0):
    R = _RefLib.get()
    N = 2 * modes - 1
    H = np.empty((N, N))
    R.check(R.h_dense(modes, period, _ptr(H)))
    return H


def ref_oracle_h_dense(modes, period=1.0):
    R = _RefLib.get()
    N = 2 * modes - 1
    H = np.empty((N, N))
    R.check(R.oracle_h_dense(modes, period, _ptr(H)))
    return H


def ref_apply_h(modes, period, series):
    R = _RefLib.get()
    s = _f64(series)
    out = np.empty_like(s)
    N = 2 * modes - 1
    R.check(R.apply_h(modes, period, _ptr(s), _ptr(out), s.size // N))
    return out


class RefCtx:
    """Reference solver objects for one mesh/basis: geometry, pattern,
    TangentOperator, BCs, AssemblyConfig."""

    def __init__(self, rmesh: RefMesh, modes: int, period: float = 1.0, rho=1.06, mu=0.04):
        self.R = _RefLib.get()
        self.rmesh = rmesh
        self.N = 2 * modes - 1
        self.nn = rmesh.sizes()[0]
        self.h = self.R.ctx_create(rmesh.h, modes, period, rho, mu)
        if not self.h:
            raise OracleError(self.R.last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.R.ctx_destroy(self.h)
            self.h = None

    @property
    def n(self):
        return self.nn * 4 * self.N

    def set_bcs(self, dirichlet_g=None, neumann=(), beta=0.2):
        g = None if dirichlet_g is None else _f64(dirichlet_g)
        pidx = np.array([p for p, _ in neumann], np.int32)
        hh = _f64(np.concatenate([np.asarray(h, float) for _, h in neumann])) if neumann else np.zeros(0)
        self.R.check(self.R.set_bcs(self.h, _ptr(g), len(pidx), _ptr(pidx), _ptr(hh), beta))

    def set_cfg(self, tau_mode=0, pseudo_dt=float("inf"), c1=1.5, backflow_tangent=False):
        pdt = pseudo_dt if np.isfinite(pseudo_dt) else 0.0
        self.R.check(self.R.set_cfg(self.h, tau_mode, pdt, c1, int(backflow_tangent)))

    def residual(self, state, threads=1):
        s = _f64(state)
        r = np.empty(self.n)
        self.R.check(self.R.residual(self.h, _ptr(s), threads, _ptr(r)))
        return r

    def oracle_residual(self, state):
        s = _f64(state)
        r = np.empty(self.n)
        self.R.check(self.R.oracle_residual(self.h, _ptr(s), _ptr(r)))
        return r

    def frozen_residual(self, state, coeff_state):
        s, c = _f64(state), _f64(coeff_state)
        r = np.empty(self.n)
        self.R.check(self.R.frozen_residual(self.h, _ptr(s), _ptr(c), _ptr(r)))
        return r

    def tangent(self, state):
        s = _f64(state)
        p = np.empty(self.R.pvals_size(self.h))
        self.R.check(self.R.tangent(self.h, _ptr(s), _ptr(p)))
        return p

    def set_pvals(self, p):
        self.R.check(self.R.set_pvals(self.h, _ptr(_f64(p))))

    def mass(self):
        nnz = self.R.pvals_size(self.h) // (8 * self.N)
        m = np.empty(nnz)
        self.R.check(self.R.mass(self.h, _ptr(m)))
        return m

    def matvec(self, y, threads=1):
        v = _f64(y)
        o = np.empty_like(v)
        self.R.check(self.R.matvec(self.h, _ptr(v), _ptr(o), threads))
        return o

    def bsr_matvec(self, y, threads=1):
        v = _f64(y)
        o = np.empty_like(v)
        self.R.check(self.R.bsr_matvec(self.h, _ptr(v), _ptr(o), threads))
        return o

    def jacobi(self):
        inv = np.empty(self.n)
        deg = C.c_int()
        self.R.check(self.R.jacobi(self.h, _ptr(inv), C.byref(deg)))
        return inv, deg.value

    def gmres(self, rhs, inv_diag, restart=200, max_iters=1000, tol=0.03, threads=1):
        b, inv = _f64(rhs), _f64(inv_diag)
        x = np.empty_like(b)
        it, st, hl = C.c_int(), C.c_int(), C.c_int()
        rr = C.c_double()
        hist = np.empty(max_iters + 2)
        self.R.check(self.R.gmres(self.h, _ptr(b), _ptr(inv), restart, max_iters, tol, threads, _ptr(x),
                                  C.byref(it), C.byref(rr), C.byref(st), _ptr(hist), len(hist), C.byref(hl)))
        return dict(x=x, iterations=it.value, relative_residual=rr.value, status=st.value,
                    history=hist[: min(hl.value, len(hist))].copy())

    def install_dirichlet(self, state):
        s = _f64(state).copy()
        self.R.check(self.R.install_dirichlet(self.h, _ptr(s)))
        return s

    def initial_pressure(self):
        return self.R.initial_pressure(self.h)

    def suggest_pseudo_dt(self):
        return self.R.suggest_dt(self.h)

    def dense_tangent(self, state):
        s = _f64(state)
        d = np.empty((self.n, self.n))
        self.R.check(self.R.dense_tangent(self.h, _ptr(s), _ptr(d)))
        return d

    def solve(self, pseudo_dt=0.0, orders=3.0, max_newton=60, restart=200, max_iters=1000, tol=0.03,
              tau_mode=0, threads=1):
        state = np.empty(self.n)
        conv = C.c_int()
        cap = max_newton + 2
        ll = C.c_int()
        res, rel = np.zeros(cap), np.zeros(cap)
        lin = np.zeros(cap, np.int32)
        sc = np.zeros(5)
        self.R.check(self.R.solve(self.h, pseudo_dt, orders, max_newton, restart, max_iters, tol, tau_mode,
                                  threads, _ptr(state), C.byref(conv), cap, C.byref(ll), _ptr(res), _ptr(rel),
                                  _ptr(lin), _ptr(sc)))
        k = min(ll.value, cap)
        return dict(state=state, converged=bool(conv.value), res=res[:k], rel=rel[:k], linear=lin[:k],
                    pseudo_dt=sc[0], cfl=sc[1], assembly_seconds=sc[2], linear_seconds=sc[3],
                    total_seconds=sc[4])


    def solve_time(self, dirichlet, period, steps=500, cycles=4, rho_inf=0.2, orders=3.0, max_newton=8,
                   restart=200, max_iters=1000, tol=0.03, steady=False, threads=1):
        """Reference solve_time (time_solver.cpp:269-485).  `dirichlet(t) -> (g, gdot)`
        (node*3+i arrays).  Returns the last cycle's snapshots and the TimeSolution scalars."""
        nn = self.n // (4 * self.N)
        cb = time_dirichlet_callback(dirichlet, nn)
        nsnap = 1 if steady else steps + 1
        u = np.empty(nsnap * nn * 3)
        p = np.empty(nsnap * nn)
        sc = np.zeros(5)
        self.R.check(self.R.solve_time(self.h, period, steps, cycles, rho_inf, orders, max_newton, restart,
                                       max_iters, tol, int(steady), threads, C.cast(cb, _vp), None, _ptr(u),
                                       _ptr(p), _ptr(sc)))
        return dict(u=u.reshape(nsnap, nn * 3), p=p.reshape(nsnap, nn), cycle_change=sc[0],
                    total_seconds=sc[1], omega_hat_last=sc[2], total_steps=int(sc[3]),
                    total_newton_iters=int(sc[4]))


TIME_DIRICHLET_FN = C.CFUNCTYPE(None, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)


def time_dirichlet_callback(fn, nn):
    """C callback (t, g*, gdot*, user) around a Python `fn(t) -> (g, gdot)`."""
    def cb(t, g, gd, _user):
        a, b = fn(t)
        C.memmove(g, _f64(a).ctypes.data, nn * 3 * 8)
        C.memmove(gd, _f64(b).ctypes.data, nn * 3 * 8)
    return TIME_DIRICHLET_FN(cb)


def ref_context(prob, tau_mode=0, pseudo_dt=float("inf")):
    """RefMesh + RefCtx for a paper_2411_14315_b200.cases.Problem."""
    rm = RefMesh.from_mesh(prob.mesh)
    ctx = RefCtx(rm, prob.modes, prob.period, prob.rho, prob.mu)
    ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
    ctx.set_cfg(tau_mode, pseudo_dt)
    return ctx


# ------------------------------------------------------------------ restatement

class _Problem(C.Structure):
    _fields_ = [
        ("nn", _i), ("ne", _i), ("conn", _vp), ("geom", _vp), ("dirichlet", _vp), ("N", _i), ("H", _vp),
        ("rho", _d), ("mu", _d), ("tau_mode", _i), ("pseudo_dt", _d), ("pseudo_c1", _d),
        ("backflow_in_tangent", _i), ("nfac", _i), ("fac", _vp), ("fnormal", _vp), ("farea", _vp),
        ("fbc", _vp), ("h", _vp), ("beta", _d), ("resistance", _vp),
    ]


class _KCfg(C.Structure):
    _fields_ = [("restart", _i), ("max_iters", _i), ("tolerance", _d)]


class _KRes(C.Structure):
    _fields_ = [("iterations", _i), ("relative_residual", _d), ("status", _i), ("history_len", _i)]


class Restated:
    """The plain-C restatement bound to one problem (mesh + basis + BCs + cfg)."""

    def __init__(self, prob, tau_mode=0, pseudo_dt=float("inf"), pseudo_c1=1.5, backflow_tangent=False,
                 geometry=None, resistance=None):
        """resistance: {patch_index: R} for resistance outlets (Neumann patches)."""
        if not os.path.exists(ORACLE_SO):
            raise OracleError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        self.L = L
        _sig(L, "hbo_h_dense", None, [_i, _d, _vp])
        _sig(L, "hbo_geometry", _i, [_i, _vp, _i, _vp, _vp])
        _sig(L, "hbo_pattern", _i, [_i, _i, _vp, _vp, _vp])
        _sig(L, "hbo_residual", _i, [_vp, _vp, _vp])
        _sig(L, "hbo_tangent", _i, [_vp, _vp, _vp, _vp, _vp])
        _sig(L, "hbo_residual_rows", _i, [_vp, _vp, _i, _vp, _vp])
        _sig(L, "hbo_tangent_rows", _i, [_vp, _vp, _vp, _vp, _i, _vp, _vp])
        _sig(L, "hbo_tangent_matvec_rows", _i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp])
        _sig(L, "hbo_mass", None, [_vp, _vp, _vp, _vp])
        _sig(L, "hbo_bsr_matvec", None, [_i, _i, _vp, _vp, _vp, _vp, _vp])
        _sig(L, "hbo_tangent_matvec", None, [_vp, _vp, _vp, _vp, _vp, _vp, _vp])
        _sig(L, "hbo_jacobi", _i, [_i, _i, _vp, _vp, _vp, _vp])
        _sig(L, "hbo_gmres_tangent", None, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp])
        _sig(L, "hbo_time_residual", None, [_vp, _vp, _vp, _vp, _d, _vp])
        _sig(L, "hbo_time_tangent", None, [_vp, _vp, _vp, _vp, _d, _d, _d, _vp])
        m = prob.mesh
        self.prob = prob
        self.N = prob.N
        self.nn = m.num_nodes
        self.conn = np.ascontiguousarray(m.conn, np.int32)
        if geometry is None:
            geometry = restated_geometry(m.xyz, self.conn)
        self.geom = _f64(geometry)
        self.dm = np.ascontiguousarray(m.dirichlet, np.uint8)
        self.H = restated_h_dense(prob.modes, prob.period)
        facs, nrms, areas, fbc, hs = [], [], [], [], []
        for k, (pidx, h) in enumerate(prob.neumann):
            p = m.patches[pidx]
            facs.append(p.facets)
            nrms.append(p.normals)
            areas.append(p.areas)
            fbc.append(np.full(len(p.facets), k, np.int32))
            hs.append(np.asarray(h, float))
        self.fac = np.ascontiguousarray(np.concatenate(facs) if facs else np.zeros((0, 3)), np.int32)
        self.fn = _f64(np.concatenate(nrms) if nrms else np.zeros((0, 3)))
        self.fa = _f64(np.concatenate(areas) if areas else np.zeros(0))
        self.fbc = np.ascontiguousarray(np.concatenate(fbc) if fbc else np.zeros(0), np.int32)
        self.hh = _f64(np.concatenate(hs) if hs else np.zeros(0))
        res = dict(resistance or {})
        self.res = _f64([float(res.get(pidx, 0.0)) for pidx, _ in prob.neumann]) if res else None
        self.p = _Problem(self.nn, m.num_elements, _ptr(self.conn), _ptr(self.geom), _ptr(self.dm), self.N,
                          _ptr(self.H), prob.rho, prob.mu, tau_mode,
                          pseudo_dt if np.isfinite(pseudo_dt) else 0.0, pseudo_c1, int(backflow_tangent),
                          len(self.fa), _ptr(self.fac), _ptr(self.fn), _ptr(self.fa), _ptr(self.fbc),
                          _ptr(self.hh), prob.backflow_beta, _ptr(self.res))
        self.row_ptr, self.col_idx = restated_pattern(self.nn, self.conn)

    @property
    def n(self):
        return self.nn * 4 * self.N

    def residual(self, state):
        s = _f64(state)
        r = np.empty(self.n)
        if self.L.hbo_residual(C.byref(self.p), _ptr(s), _ptr(r)):
            raise ArithmeticError("singular stabilization parameter")
        return r

    def tangent(self, state):
        s = _f64(state)
        v = np.empty(len(self.col_idx) * 8 * self.N)
        if self.L.hbo_tangent(C.byref(self.p), _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(s), _ptr(v)):
            raise ArithmeticError("singular stabilization parameter")
        return v

    def _rows_status(self, st):
        if st == -1:
            raise ArithmeticError("singular stabilization parameter")
        if st:
            raise OracleError(f"row subset: status {st} (rows must be distinct and in range)")

    def residual_rows(self, state, rows):
        """Residual rows of the listed nodes, (len(rows), 4, N); bit-identical to
        the corresponding rows of residual()."""
        s = _f64(state)
        rows = np.ascontiguousarray(rows, np.int32)
        r = np.empty(len(rows) * 4 * self.N)
        self._rows_status(self.L.hbo_residual_rows(C.byref(self.p), _ptr(s), len(rows), _ptr(rows), _ptr(r)))
        return r.reshape(len(rows), 4, self.N)

    def tangent_rows(self, state, rows):
        """P block rows of the listed nodes: the segments
        vals[row_ptr[A]*8N : row_ptr[A+1]*8N] concatenated in list order."""
        s = _f64(state)
        rows = np.ascontiguousarray(rows, np.int32)
        tot = int(np.sum(self.row_ptr[rows + 1] - self.row_ptr[rows])) * 8 * self.N
        v = np.empty(tot)
        self._rows_status(self.L.hbo_tangent_rows(C.byref(self.p), _ptr(self.row_ptr), _ptr(self.col_idx),
                                                  _ptr(s), len(rows), _ptr(rows), _ptr(v)))
        return v

    def matvec_rows(self, row_vals, mass, y, rows):
        """TangentOperator::matvec rows of the listed nodes from their P
        segments (tangent_rows layout), the full mass and the full y."""
        rv, m, yy = _f64(row_vals), _f64(mass), _f64(y)
        rows = np.ascontiguousarray(rows, np.int32)
        o = np.empty(len(rows) * 4 * self.N)
        self._rows_status(self.L.hbo_tangent_matvec_rows(C.byref(self.p), _ptr(self.row_ptr), _ptr(self.col_idx),
                                                         _ptr(rv), _ptr(m), _ptr(yy), len(rows), _ptr(rows),
                                                         _ptr(o)))
        return o.reshape(len(rows), 4, self.N)

    def time_residual(self, u, udot, p, omega_hat):
        """time_solver.cpp:58-166 (u, udot node*3+i, p node) -> r node*4+c"""
        u, ud, pp = _f64(u), _f64(udot), _f64(p)
        r = np.empty(self.nn * 4)
        self.L.hbo_time_residual(C.byref(self.p), _ptr(u), _ptr(ud), _ptr(pp), float(omega_hat), _ptr(r))
        return r

    def time_tangent(self, u, omega_hat, am, fg):
        """time_solver.cpp:172-254 -> N = 1 BSR values (blk*8+slot)"""
        u = _f64(u)
        v = np.empty(len(self.col_idx) * 8)
        self.L.hbo_time_tangent(C.byref(self.p), _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(u),
                                float(omega_hat), float(am), float(fg), _ptr(v))
        return v

    def mass(self):
        m = np.empty(len(self.col_idx))
        self.L.hbo_mass(C.byref(self.p), _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(m))
        return m

    def bsr_matvec(self, vals, y):
        v, yy = _f64(vals), _f64(y)
        o = np.empty(self.n)
        self.L.hbo_bsr_matvec(self.nn, self.N, _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(v), _ptr(yy), _ptr(o))
        return o

    def matvec(self, vals, mass, y):
        v, m, yy = _f64(vals), _f64(mass), _f64(y)
        o = np.empty(self.n)
        self.L.hbo_tangent_matvec(C.byref(self.p), _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(v), _ptr(m),
                                  _ptr(yy), _ptr(o))
        return o

    def jacobi(self, vals):
        v = _f64(vals)
        inv = np.empty(self.n)
        deg = self.L.hbo_jacobi(self.nn, self.N, _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(v), _ptr(inv))
        return inv, deg

    def gmres(self, vals, mass, rhs, inv_diag, restart=200, max_iters=1000, tol=0.03):
        v, m, b, inv = _f64(vals), _f64(mass), _f64(rhs), _f64(inv_diag)
        x = np.empty(self.n)
        hist = np.empty(max_iters + 2)
        cfg = _KCfg(restart, max_iters, tol)
        res = _KRes()
        self.L.hbo_gmres_tangent(C.byref(self.p), _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(v), _ptr(m),
                                 _ptr(b), _ptr(inv), C.byref(cfg), _ptr(x), C.byref(res), _ptr(hist))
        return dict(x=x, iterations=res.iterations, relative_residual=res.relative_residual,
                    status=res.status, history=hist[: res.history_len].copy())


def _olib():
    L = C.CDLL(ORACLE_SO)
    _sig(L, "hbo_h_dense", None, [_i, _d, _vp])
    _sig(L, "hbo_geometry", _i, [_i, _vp, _i, _vp, _vp])
    _sig(L, "hbo_pattern", _i, [_i, _i, _vp, _vp, _vp])
    return L


def restated_h_dense(modes, period=1.0):
    N = 2 * modes - 1
    H = np.empty((N, N))
    _olib().hbo_h_dense(modes, period, _ptr(H))
    return H


def restated_geometry(xyz, conn):
    xyz, conn = _f64(xyz), np.ascontiguousarray(conn, np.int32)
    g = np.empty((conn.shape[0], 22))
    if _olib().hbo_geometry(xyz.shape[0], _ptr(xyz), conn.shape[0], _ptr(conn), _ptr(g)):
        raise OracleError("degenerate element")
    return g


def restated_pattern(nn, conn):
    conn = np.ascontiguousarray(conn, np.int32)
    L = _olib()
    rp = np.empty(nn + 1, np.int32)
    nnz = L.hbo_pattern(nn, conn.shape[0], _ptr(conn), _ptr(rp), None)
    ci = np.empty(nnz, np.int32)
    L.hbo_pattern(nn, conn.shape[0], _ptr(conn), _ptr(rp), _ptr(ci))
    return rp, ci
