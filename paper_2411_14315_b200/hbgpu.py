"""Python host mirror of the reference hot-path interface over the C ABI.

The reference (C++, /root/reference/proj) exposes the hot path as
`assemble_residual`, `assemble_tangent`, `assemble_mass`
(include/hbflow/assembly.hpp:129-146), `TangentOperator::matvec`,
`jacobi_preconditioner`, `gmres_solve` (include/hbflow/linalg.hpp:64-115) and
`solve_harmonic` (include/hbflow/hb_solver.hpp:70-72).  This module binds the
same operations, with the same argument meaning, layouts and error
behaviour, to libhbgpu.so (include/hbgpu.h) through ctypes.  It is plumbing:
all compute runs in the CUDA library; there is no CPU fallback and import
fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from .mesh import GeometryError, Mesh, ParseError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HBGPU_LIB") or os.path.join(_HERE, "libhbgpu.so")


class StagnationError(RuntimeError):
    """GMRES made no progress over a restart cycle (errors.hpp:31-36)."""


class DivergenceError(RuntimeError):
    """Nonlinear solve blew up (errors.hpp:22-29)."""


class CudaError(RuntimeError):
    pass


_ERRORS = {
    1: ValueError,  # std::invalid_argument
    2: ArithmeticError,  # std::domain_error (singular tau)
    3: GeometryError,
    4: ParseError,
    5: StagnationError,
    6: DivergenceError,
    7: CudaError,
    8: MemoryError,
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the HB-GLS path has no CPU fallback)"
        )
    return C.CDLL(LIB_PATH)


_lib = _load()

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


class _MeshDesc(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int),
        ("num_elements", C.c_int),
        ("xyz", _vp),
        ("conn", _vp),
        ("geometry", _vp),
        ("dirichlet", _vp),
        ("num_patches", C.c_int),
        ("patch_kind", _vp),
        ("patch_num_facets", _vp),
        ("facets", _vp),
        ("normals", _vp),
        ("areas", _vp),
    ]


class _KrylovCfg(C.Structure):
    _fields_ = [("restart", C.c_int), ("max_iters", C.c_int), ("tolerance", C.c_double)]


class _KrylovRes(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("relative_residual", C.c_double),
        ("status", C.c_int),
        ("history_len", C.c_int),
        ("reorthogonalizations", C.c_int),
    ]


class _SolverCfg(C.Structure):
    _fields_ = [
        ("pseudo_dt", C.c_double),
        ("newton_tol_orders", C.c_double),
        ("max_newton_iters", C.c_int),
        ("krylov", _KrylovCfg),
        ("tau_mode", C.c_int),
        ("backflow_in_tangent", C.c_int),
        ("divergence_ratio", C.c_double),
    ]


class _SolveInfo(C.Structure):
    _fields_ = [
        ("entries", C.c_int),
        ("converged", C.c_int),
        ("pseudo_dt", C.c_double),
        ("cfl", C.c_double),
        ("assembly_seconds", C.c_double),
        ("linear_seconds", C.c_double),
        ("total_seconds", C.c_double),
    ]


class _TimeCfg(C.Structure):
    _fields_ = [
        ("steps_per_cycle", C.c_int),
        ("cycles", C.c_int),
        ("rho_inf", C.c_double),
        ("newton_tol_orders", C.c_double),
        ("max_newton_iters", C.c_int),
        ("krylov", _KrylovCfg),
        ("steady", C.c_int),
        ("initial_pressure", C.c_double),
    ]


class _TimeResult(C.Structure):
    _fields_ = [
        ("cycle_change", C.c_double),
        ("total_seconds", C.c_double),
        ("total_steps", C.c_int),
        ("total_newton_iters", C.c_int),
        ("omega_hat_last", C.c_double),
    ]


# TimeDirichletFn (cases.hpp:132-133): (t, g*, gdot*, user)
TimeDirichletFn = C.CFUNCTYPE(None, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_create = _sig("hbgpu_create", _vp, [C.POINTER(_MeshDesc), _ip])
_destroy = _sig("hbgpu_destroy", None, [_vp])
_last_error = _sig("hbgpu_last_error", C.c_char_p, [_vp])
_create_error = _sig("hbgpu_create_error", C.c_char_p, [])
_stream = _sig("hbgpu_stream", _vp, [_vp])
_sync = _sig("hbgpu_synchronize", C.c_int, [_vp])
_set_basis = _sig("hbgpu_set_basis", C.c_int, [_vp, C.c_int, C.c_double])
_set_fluid = _sig("hbgpu_set_fluid", C.c_int, [_vp, C.c_double, C.c_double])
_set_bcs = _sig("hbgpu_set_bcs", C.c_int, [_vp, _vp, C.c_int, _vp, _vp, C.c_double])
_set_cfg = _sig("hbgpu_set_assembly_config", C.c_int, [_vp, C.c_int, C.c_double, C.c_double, C.c_int])
_sizes = _sig("hbgpu_sizes", C.c_int, [_vp, _ip, _ip, _ip, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)])
_get_pattern = _sig("hbgpu_get_pattern", C.c_int, [_vp, _vp, _vp])
_get_geometry = _sig("hbgpu_get_geometry", C.c_int, [_vp, _vp])
_residual = _sig("hbgpu_assemble_residual", C.c_int, [_vp, _vp, _vp])
_assemble = _sig("hbgpu_assemble", C.c_int, [_vp, _vp, _vp])
_tangent = _sig("hbgpu_assemble_tangent", C.c_int, [_vp, _vp, _vp])
_mass = _sig("hbgpu_assemble_mass", C.c_int, [_vp, _vp])
_set_pvals = _sig("hbgpu_set_pvals", C.c_int, [_vp, _vp])
_set_mass = _sig("hbgpu_set_mass", C.c_int, [_vp, _vp])
_matvec = _sig("hbgpu_matvec", C.c_int, [_vp, _vp, _vp])
_bsr_matvec = _sig("hbgpu_bsr_matvec", C.c_int, [_vp, _vp, _vp])
_jacobi = _sig("hbgpu_jacobi", C.c_int, [_vp, _vp, _ip])
_APPLY_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double))
_gmres_apply = _sig("hbgpu_gmres_apply", C.c_int, [_vp, _APPLY_FN, _vp, C.c_longlong, _vp, _vp,
                                                   C.POINTER(_KrylovCfg), _vp, C.POINTER(_KrylovRes), _vp, C.c_int])
_gmres = _sig("hbgpu_gmres", C.c_int, [_vp, _vp, _vp, C.POINTER(_KrylovCfg), _vp, C.POINTER(_KrylovRes), _vp, C.c_int])
_residual_dev = _sig("hbgpu_assemble_residual_dev", C.c_int, [_vp, _vp, _vp])
_tangent_dev = _sig("hbgpu_assemble_tangent_dev", C.c_int, [_vp, _vp])
_assemble_dev = _sig("hbgpu_assemble_dev", C.c_int, [_vp, _vp, _vp])
_matvec_dev = _sig("hbgpu_matvec_dev", C.c_int, [_vp, _vp, _vp])
_bsr_matvec_dev = _sig("hbgpu_bsr_matvec_dev", C.c_int, [_vp, _vp, _vp])
_jacobi_dev = _sig("hbgpu_jacobi_dev", C.c_int, [_vp, _ip])
_gmres_dev = _sig("hbgpu_gmres_dev", C.c_int, [_vp, _vp, C.POINTER(_KrylovCfg), _vp, C.POINTER(_KrylovRes), _vp, C.c_int])
_pvals_dev = _sig("hbgpu_pvals_dev", _vp, [_vp])
_get_pvals = _sig("hbgpu_get_pvals", C.c_int, [_vp, _vp])
_get_pvals_rows = _sig("hbgpu_get_pvals_rows", C.c_int, [_vp, C.c_int, _vp, _vp])
_set_resistance = _sig("hbgpu_set_resistance", C.c_int, [_vp, C.c_int, _vp, _vp])
_time_residual = _sig("hbgpu_time_residual", C.c_int, [_vp, _vp, _vp, _vp, C.c_double, _vp])
_time_tangent = _sig("hbgpu_time_tangent", C.c_int, [_vp, _vp, C.c_double, C.c_double, C.c_double, _vp])
_solve_time = _sig("hbgpu_solve_time", C.c_int,
                   [_vp, C.POINTER(_TimeCfg), C.c_double, TimeDirichletFn, _vp, _vp, _vp, C.POINTER(_TimeResult)])
_solve = _sig(
    "hbgpu_solve_harmonic",
    C.c_int,
    [_vp, C.POINTER(_SolverCfg), _vp, C.POINTER(_SolveInfo), C.c_int, _vp, _vp, _vp, _vp, _vp],
)

def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class KrylovConfig:
    """linalg.hpp:86-90"""

    restart: int = 200
    max_iters: int = 1000
    tolerance: float = 0.03


@dataclass
class KrylovResult:
    """linalg.hpp:94-100; status 0 Converged, 1 MaxIterations, 2 Stagnated"""

    x: np.ndarray
    iterations: int
    relative_residual: float
    status: int
    history: np.ndarray


@dataclass
class SolverConfig:
    """hb_solver.hpp:12-23"""

    pseudo_dt: float = 0.0
    newton_tol_orders: float = 3.0
    max_newton_iters: int = 60
    krylov: KrylovConfig = field(default_factory=KrylovConfig)
    tau_mode: int = 0
    backflow_in_tangent: bool = False
    divergence_ratio: float = 1e3


@dataclass
class ConvergenceLog:
    """hb_solver.hpp:25-38; to_csv matches hb_solver.cpp:74-84"""

    iters: np.ndarray
    res: np.ndarray
    res_rel: np.ndarray
    linear_iters: np.ndarray
    seconds: np.ndarray
    converged: bool

    def to_csv(self) -> str:
        lines = ["iter,res,res_rel,linear_iters,seconds"]
        for k in range(len(self.iters)):
            lines.append(
                "%d,%.17g,%.17g,%d,%.6f"
                % (self.iters[k], self.res[k], self.res_rel[k], self.linear_iters[k], self.seconds[k])
            )
        return "\n".join(lines) + "\n"


@dataclass
class TimeSolverConfig:
    """time_solver.hpp:11-22"""

    steps_per_cycle: int = 500
    cycles: int = 4
    rho_inf: float = 0.2
    newton_tol_orders: float = 3.0
    max_newton_iters: int = 8
    krylov: KrylovConfig = field(default_factory=KrylovConfig)
    steady: bool = False
    initial_pressure: float = float("nan")  # NaN: from the context's Neumann data


@dataclass
class TimeSolution:
    """time_solver.hpp:24-49: the last cycle's snapshots u[(steps+1), nodes*3],
    p[(steps+1), nodes] (one snapshot when steady) and the run scalars."""

    u: np.ndarray
    p: np.ndarray
    period: float
    cycle_change: float
    total_seconds: float
    total_steps: int
    total_newton_iters: int
    omega_hat_last: float


@dataclass
class HbSolution:
    """hb_solver.hpp:40-48"""

    state: np.ndarray
    log: ConvergenceLog
    pseudo_dt: float
    cfl: float
    assembly_seconds: float
    linear_seconds: float
    total_seconds: float


class GpuContext:
    """Device context: mesh, pattern and work buffers of one solve.

    Mirrors the reference objects the hot path reads: Mesh + geometry
    (mesh.hpp), SpectralBasis/SpectralOperators (spectral.hpp),
    FluidProperties / BoundaryConditionSet / AssemblyConfig (assembly.hpp) and
    the TangentOperator (linalg.hpp:64-76) whose P, mass and Jacobi vector stay
    on the device.
    """

    def __init__(self, mesh: Mesh, geometry: np.ndarray | None = None):
        if mesh.dirichlet is None:
            mesh.finalize()
        self.mesh = mesh
        self._keep = []
        xyz = _f64(mesh.xyz)
        conn = np.ascontiguousarray(mesh.conn, dtype=np.int32)
        dmask = np.ascontiguousarray(mesh.dirichlet, dtype=np.uint8)
        kinds = np.array([p.kind for p in mesh.patches], dtype=np.int32)
        nf = np.array([len(p.facets) for p in mesh.patches], dtype=np.int32)
        if mesh.patches:
            facets = np.ascontiguousarray(np.concatenate([p.facets for p in mesh.patches]), dtype=np.int32)
            normals = _f64(np.concatenate([p.normals for p in mesh.patches]))
            areas = _f64(np.concatenate([p.areas for p in mesh.patches]))
        else:
            facets = np.zeros((0, 3), np.int32)
            normals = np.zeros((0, 3))
            areas = np.zeros(0)
        geo = None if geometry is None else _f64(geometry)
        self._keep = [xyz, conn, dmask, kinds, nf, facets, normals, areas, geo]
        d = _MeshDesc(
            mesh.num_nodes, mesh.num_elements, _ptr(xyz), _ptr(conn), _ptr(geo), _ptr(dmask),
            len(mesh.patches), _ptr(kinds), _ptr(nf), _ptr(facets), _ptr(normals), _ptr(areas),
        )
        st = C.c_int(0)
        h = _create(C.byref(d), C.byref(st))
        if not h:
            raise _ERRORS.get(st.value, RuntimeError)(_create_error().decode())
        self._h = h
        self.N = 0
        self.M = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _destroy is not None:  # module globals may be gone at interpreter exit
            _destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    # ------------------------------------------------------------ plumbing
    def _check(self, status: int):
        if status != 0:
            raise _ERRORS.get(status, RuntimeError)(_last_error(self._h).decode())

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return _stream(self._h)

    def synchronize(self):
        self._check(_sync(self._h))

    def sizes(self):
        nn, ne, N = C.c_int(), C.c_int(), C.c_int()
        nnz, sl = C.c_longlong(), C.c_longlong()
        _sizes(self._h, C.byref(nn), C.byref(ne), C.byref(N), C.byref(nnz), C.byref(sl))
        return nn.value, ne.value, N.value, nnz.value, sl.value

    @property
    def nnz(self) -> int:
        return self.sizes()[3]

    @property
    def state_len(self) -> int:
        return self.sizes()[4]

    # ------------------------------------------------------------ setup
    def set_basis(self, modes: int, period: float = 1.0):
        self._check(_set_basis(self._h, int(modes), float(period)))
        self.M, self.N = int(modes), 2 * int(modes) - 1
        self.period = float(period)

    def set_fluid(self, rho: float = 1.06, mu: float = 0.04):
        self._check(_set_fluid(self._h, float(rho), float(mu)))

    def set_bcs(self, dirichlet_g=None, neumann=(), backflow_beta: float = 0.2):
        """neumann: sequence of (patch_index, h[N])."""
        g = None if dirichlet_g is None else _f64(dirichlet_g)
        pidx = np.array([p for p, _ in neumann], dtype=np.int32)
        hh = _f64(np.array([np.asarray(h, dtype=np.float64) for _, h in neumann]).reshape(-1)) if neumann else np.zeros(0)
        self._check(_set_bcs(self._h, _ptr(g), len(pidx), _ptr(pidx), _ptr(hh), float(backflow_beta)))

    def pvals(self) -> np.ndarray:
        """The current P values (after assemble / assemble_tangent / set_pvals)."""
        v = np.empty(self.nnz * 8 * self.N)
        self._check(_get_pvals(self._h, _ptr(v)))
        return v

    def pvals_rows(self, rows, row_ptr=None) -> np.ndarray:
        """P block rows of the listed nodes, concatenated in list order
        (hbgpu_get_pvals_rows): a sample of P without reading all of it."""
        rows = np.ascontiguousarray(rows, np.int32)
        if row_ptr is None:
            row_ptr = self.pattern()[0]
        tot = int(np.sum(row_ptr[rows + 1].astype(np.int64) - row_ptr[rows])) * 8 * self.N
        v = np.empty(tot)
        self._check(_get_pvals_rows(self._h, len(rows), _ptr(rows), _ptr(v)))
        return v

    def set_resistance(self, resistance: dict):
        """{neumann patch index: R} resistance outlets (hbgpu_set_resistance)."""
        pk = np.array(list(resistance.keys()), np.int32)
        rv = _f64(list(resistance.values()))
        self._check(_set_resistance(self._h, len(pk), _ptr(pk), _ptr(rv)))

    def set_assembly_config(self, tau_mode: int = 0, pseudo_dt: float = float("inf"),
                            pseudo_c1: float = 1.5, backflow_in_tangent: bool = False):
        pdt = float(pseudo_dt) if np.isfinite(pseudo_dt) else 0.0
        self._check(_set_cfg(self._h, int(tau_mode), pdt, float(pseudo_c1), int(bool(backflow_in_tangent))))

    def pattern(self):
        nn, _, _, nnz, _ = self.sizes()
        rp = np.empty(nn + 1, np.int32)
        ci = np.empty(nnz, np.int32)
        self._check(_get_pattern(self._h, _ptr(rp), _ptr(ci)))
        return rp, ci

    def geometry(self):
        g = np.empty((self.mesh.num_elements, 22))
        self._check(_get_geometry(self._h, _ptr(g)))
        return g

    # ------------------------------------------------------------ drop-ins
    def _vec_in(self, v) -> np.ndarray:
        v = _f64(v).reshape(-1)
        if v.size != self.state_len:
            raise ValueError("vector size mismatch")
        return v

    def assemble_residual(self, state) -> np.ndarray:
        s = self._vec_in(state)
        r = np.empty_like(s)
        self._check(_residual(self._h, _ptr(s), _ptr(r)))
        return r

    def assemble(self, state) -> np.ndarray:
        """Residual (returned) and tangent (kept on the device) of one host
        state with a single upload (hbgpu_assemble)."""
        s = self._vec_in(state)
        r = np.empty_like(s)
        self._check(_assemble(self._h, _ptr(s), _ptr(r)))
        return r

    def assemble_tangent(self, state, download: bool = True):
        s = self._vec_in(state)
        out = np.empty(self.nnz * 8 * self.N) if download else None
        self._check(_tangent(self._h, _ptr(s), _ptr(out)))
        return out

    def assemble_mass(self) -> np.ndarray:
        m = np.empty(self.nnz)
        self._check(_mass(self._h, _ptr(m)))
        return m

    def set_pvals(self, pvals):
        p = _f64(pvals).reshape(-1)
        if p.size != self.nnz * 8 * self.N:
            raise ValueError("P values size mismatch")
        self._check(_set_pvals(self._h, _ptr(p)))

    def set_mass(self, mass):
        """Replace the device node-pair mass (TangentOperator::mass)."""
        m = _f64(mass).reshape(-1)
        if m.size != self.nnz:
            raise ValueError("mass size mismatch")
        self._check(_set_mass(self._h, _ptr(m)))

    def matvec(self, y) -> np.ndarray:
        v = self._vec_in(y)
        o = np.empty_like(v)
        self._check(_matvec(self._h, _ptr(v), _ptr(o)))
        return o

    def bsr_matvec(self, y) -> np.ndarray:
        v = self._vec_in(y)
        o = np.empty_like(v)
        self._check(_bsr_matvec(self._h, _ptr(v), _ptr(o)))
        return o

    def jacobi(self):
        inv = np.empty(self.state_len)
        deg = C.c_int(0)
        self._check(_jacobi(self._h, _ptr(inv), C.byref(deg)))
        return inv, deg.value

    def gmres_apply(self, apply, rhs, inv_diag, cfg: KrylovConfig | None = None) -> KrylovResult:
        """gmres_solve(apply, rhs, inv_diag, cfg) (linalg.hpp:107-109): the
        generic overload with a host operator `apply(y) -> A y` (numpy arrays);
        Krylov basis and orthogonalisation on the device."""
        cfg = cfg or KrylovConfig()
        b = _f64(rhs).reshape(-1)
        inv = _f64(inv_diag).reshape(-1)
        n = b.size
        if inv.size != n:
            raise ValueError("gmres_apply: size mismatch")

        def cb(_user, y, out):
            yv = np.ctypeslib.as_array(y, shape=(n,))
            ov = np.ctypeslib.as_array(out, shape=(n,))
            ov[:] = apply(yv.copy())

        fn = _APPLY_FN(cb)
        x = np.empty(n)
        res = _KrylovRes()
        hist = np.empty(cfg.max_iters + 2)
        kc = _KrylovCfg(cfg.restart, cfg.max_iters, cfg.tolerance)
        self._check(_gmres_apply(self._h, fn, None, n, _ptr(b), _ptr(inv), C.byref(kc), _ptr(x), C.byref(res),
                                 _ptr(hist), len(hist)))
        return KrylovResult(x, res.iterations, res.relative_residual, res.status, hist[: res.history_len].copy())

    def gmres(self, rhs, cfg: KrylovConfig | None = None, inv_diag=None) -> KrylovResult:
        cfg = cfg or KrylovConfig()
        b = self._vec_in(rhs)
        inv = None if inv_diag is None else self._vec_in(inv_diag)
        x = np.empty_like(b)
        hist = np.empty(cfg.max_iters + 2)
        kc = _KrylovCfg(cfg.restart, cfg.max_iters, cfg.tolerance)
        kr = _KrylovRes()
        self._check(_gmres(self._h, _ptr(b), _ptr(inv), C.byref(kc), _ptr(x), C.byref(kr), _ptr(hist), len(hist)))
        return KrylovResult(x, kr.iterations, kr.relative_residual, kr.status, hist[: kr.history_len].copy())

    # ------------------------------------------------------------ device fast path
    def assemble_residual_dev(self, d_state: int, d_r: int):
        self._check(_residual_dev(self._h, d_state, d_r))

    def assemble_tangent_dev(self, d_state: int):
        self._check(_tangent_dev(self._h, d_state))

    def assemble_dev(self, d_state: int, d_r: int):
        """Residual + tangent of one iterate (concurrent on two streams)."""
        self._check(_assemble_dev(self._h, d_state, d_r))

    def matvec_dev(self, d_y: int, d_out: int):
        self._check(_matvec_dev(self._h, d_y, d_out))

    def bsr_matvec_dev(self, d_y: int, d_out: int):
        self._check(_bsr_matvec_dev(self._h, d_y, d_out))

    def jacobi_dev(self) -> int:
        deg = C.c_int(0)
        self._check(_jacobi_dev(self._h, C.byref(deg)))
        return deg.value

    def gmres_dev(self, d_rhs: int, d_x: int, cfg: KrylovConfig | None = None):
        cfg = cfg or KrylovConfig()
        kc = _KrylovCfg(cfg.restart, cfg.max_iters, cfg.tolerance)
        kr = _KrylovRes()
        self._check(_gmres_dev(self._h, d_rhs, C.byref(kc), d_x, C.byref(kr), None, 0))
        self.last_reorthogonalizations = kr.reorthogonalizations
        return kr.iterations, kr.relative_residual, kr.status

    def pvals_dev(self) -> int:
        return _pvals_dev(self._h)

    # ------------------------------------------------------------ time solver
    def time_residual(self, u, udot, p, omega_hat: float = 0.0) -> np.ndarray:
        """time_residual (time_solver.cpp:58-166); N = 1 context."""
        u, ud, pp = _f64(u), _f64(udot), _f64(p)
        r = np.empty(self.mesh.num_nodes * 4)
        self._check(_time_residual(self._h, _ptr(u), _ptr(ud), _ptr(pp), float(omega_hat), _ptr(r)))
        return r

    def time_tangent(self, u, omega_hat: float, am: float, fg: float) -> np.ndarray:
        """time_tangent (time_solver.cpp:172-254) -> N = 1 P values (kept on device)."""
        u = _f64(u)
        v = np.empty(self.nnz * 8)
        self._check(_time_tangent(self._h, _ptr(u), float(omega_hat), float(am), float(fg), _ptr(v)))
        return v

    def solve_time(self, dirichlet, cfg: TimeSolverConfig | None = None, period: float | None = None) -> TimeSolution:
        """solve_time (time_solver.cpp:269-485) on the device.  The context must
        hold the N = 1 basis (set_basis(1, period)) and steady Neumann data;
        `dirichlet(t) -> (g, gdot)` returns node*3+i arrays (TimeDirichletFn)."""
        cfg = cfg or TimeSolverConfig()
        period = float(self.period if period is None else period)
        nn = self.mesh.num_nodes

        def cb(t, g, gd, _user):
            a, b = dirichlet(t)
            C.memmove(g, _f64(a).ctypes.data, nn * 3 * 8)
            C.memmove(gd, _f64(b).ctypes.data, nn * 3 * 8)

        fn = TimeDirichletFn(cb)
        tc = _TimeCfg(int(cfg.steps_per_cycle), int(cfg.cycles), float(cfg.rho_inf), float(cfg.newton_tol_orders),
                      int(cfg.max_newton_iters),
                      _KrylovCfg(cfg.krylov.restart, cfg.krylov.max_iters, cfg.krylov.tolerance), int(bool(cfg.steady)),
                      float(cfg.initial_pressure))
        nsnap = 1 if cfg.steady else cfg.steps_per_cycle + 1
        u = np.empty(nsnap * nn * 3)
        p = np.empty(nsnap * nn)
        res = _TimeResult()
        self._check(_solve_time(self._h, C.byref(tc), period, fn, None, _ptr(u), _ptr(p), C.byref(res)))
        return TimeSolution(u.reshape(nsnap, nn * 3), p.reshape(nsnap, nn), period, res.cycle_change,
                            res.total_seconds, res.total_steps, res.total_newton_iters, res.omega_hat_last)

    # ------------------------------------------------------------ Newton
    def solve_harmonic(self, cfg: SolverConfig | None = None) -> HbSolution:
        cfg = cfg or SolverConfig()
        sc = _SolverCfg(
            float(cfg.pseudo_dt), float(cfg.newton_tol_orders), int(cfg.max_newton_iters),
            _KrylovCfg(cfg.krylov.restart, cfg.krylov.max_iters, cfg.krylov.tolerance),
            int(cfg.tau_mode), int(bool(cfg.backflow_in_tangent)), float(cfg.divergence_ratio),
        )
        cap = cfg.max_newton_iters + 2
        it = np.zeros(cap, np.int32)
        res = np.zeros(cap)
        rel = np.zeros(cap)
        lin = np.zeros(cap, np.int32)
        sec = np.zeros(cap)
        state = np.empty(self.state_len)
        info = _SolveInfo()
        st = _solve(self._h, C.byref(sc), _ptr(state), C.byref(info), cap, _ptr(it), _ptr(res), _ptr(rel), _ptr(lin), _ptr(sec))
        k = info.entries
        log = ConvergenceLog(it[:k], res[:k], rel[:k], lin[:k], sec[:k], bool(info.converged))
        if st != 0:
            err = _ERRORS.get(st, RuntimeError)(_last_error(self._h).decode())
            err.partial_log_csv = log.to_csv()
            raise err
        return HbSolution(state, log, info.pseudo_dt, info.cfl, info.assembly_seconds,
                          info.linear_seconds, info.total_seconds)
