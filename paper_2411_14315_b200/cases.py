"""Boundary data and synthetic states for the BASELINE.json configurations.

Mirrors the reference's case plumbing where it exists: the parabolic inlet
profile and flow scaling of build_case / rebuild_spectral
(/root/reference/proj/src/cases.cpp:575-633, 710-772), zero-traction Neumann
outlets (h = -P), and the HarmonicState layout.  The inflow waveforms are the
seeded synthetic ones BASELINE.json specifies (no patient data exists here).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import DIRICHLET, NEUMANN, GeometryError, Mesh
from . import meshgen


@dataclass
class Problem:
    mesh: Mesh
    modes: int
    period: float
    rho: float
    mu: float
    dirichlet_g: np.ndarray  # nn*3*N
    neumann: list  # [(patch_index, h[N])]
    backflow_beta: float = 0.2

    @property
    def N(self) -> int:
        return 2 * self.modes - 1


def sample_times(modes: int, period: float) -> np.ndarray:
    N = 2 * modes - 1
    return period * np.arange(N) / N  # SpectralBasis::sample_time (spectral.hpp:22)


def inflow_coefficients(cfg: int, seed: int | None = None):
    """(Q0, a_k, b_k) of Q(t) = Q0 (1 + sum_k a_k cos 2 pi k t + b_k sin 2 pi k t)."""
    rng = np.random.default_rng(cfg if seed is None else seed)
    if cfg == 0:
        a = rng.uniform(-0.3, 0.3, 2)
        b = rng.uniform(-0.3, 0.3, 2)
        return 2.0, a, b
    if cfg in (1, 2):
        k = np.arange(1, 10)
        phase = rng.uniform(0.0, 2.0 * np.pi, 9)
        amp = 0.5 / k
        return 2.0, amp * np.cos(phase), amp * np.sin(phase)
    if cfg == 3:
        # coronary-like, diastole-dominant: a broad diastolic bump minus a
        # short systolic dip, 16 harmonics, each perturbed by a seeded +-10 %
        t = np.arange(4096) / 4096.0
        bump = lambda c, w: np.exp(-(((t - c + 0.5) % 1.0 - 0.5) / w) ** 2)
        f = 0.9 * bump(0.65, 0.18) - 0.45 * bump(0.12, 0.06)
        f = f - f.mean()
        c = np.fft.rfft(f) / len(t)
        k = np.arange(1, 17)
        jit = 1.0 + 0.1 * rng.standard_normal(16)
        return 1.0, 2.0 * c[k].real * jit, -2.0 * c[k].imag * jit
    raise ValueError(f"no inflow for config {cfg}")


def flow_samples(Q0: float, a, b, modes: int, period: float) -> np.ndarray:
    """Band-limited Q at the N sample times.  All harmonics used here are in
    band (k <= M-1), so truncate_signal (spectral.cpp:77-109) is exact."""
    t = sample_times(modes, period)
    q = np.ones_like(t)
    for k, (ak, bk) in enumerate(zip(a, b), start=1):
        if k > modes - 1:
            break
        q += ak * np.cos(2 * np.pi * k * t / period) + bk * np.sin(2 * np.pi * k * t / period)
    return Q0 * q


def _inlet_frame(mesh: Mesh, p):
    """inlet_frame (cases.cpp:517-563): area-weighted centroid, inward
    direction = -mean normal, in-plane axes."""
    a = p.areas
    nbar = (a[:, None] * p.normals).sum(axis=0)
    c = (a[:, None] / 3.0 * mesh.xyz[p.facets].sum(axis=1)).sum(axis=0) / a.sum()
    nl = np.linalg.norm(nbar)
    if not nl > 0:
        raise GeometryError("inlet patch has a degenerate mean normal")
    d = -nbar / nl
    trial = np.array([1.0, 0, 0]) if abs(d[0]) < 0.9 else np.array([0, 1.0, 0])
    e1 = trial - trial.dot(d) * d
    e1 /= np.linalg.norm(e1)
    e2 = np.cross(d, e1)
    return c, d, e1, e2


def parabolic_dirichlet(mesh: Mesh, inlet: int, q: np.ndarray) -> np.ndarray:
    """dirichlet_g for a ParabolicRound inlet carrying flow q[N]
    (cases.cpp:710-772 shape + integral, cases.cpp:621-631 scaling)."""
    N = len(q)
    p = mesh.patches[inlet]
    c, d, e1, e2 = _inlet_frame(mesh, p)
    other = np.zeros(mesh.num_nodes, bool)
    for k, pp in enumerate(mesh.patches):
        if k != inlet and pp.kind == DIRICHLET:
            other[pp.facets.reshape(-1)] = True
    nodes = np.unique(p.facets)
    rel = mesh.xyz[nodes] - c
    xi, eta = rel @ e1, rel @ e2
    rmax = np.sqrt(xi * xi + eta * eta).max()
    phi = np.maximum(1.0 - (xi * xi + eta * eta) / (rmax * rmax), 0.0)
    phi[other[nodes]] = 0.0
    shape = np.zeros(mesh.num_nodes)
    shape[nodes] = phi
    tri = np.array([[2 / 3, 1 / 6, 1 / 6], [1 / 6, 2 / 3, 1 / 6], [1 / 6, 1 / 6, 2 / 3]])
    integral = float((p.areas / 3.0 * (shape[p.facets] @ tri.T).sum(axis=1)).sum())
    if not integral > 0:
        raise GeometryError("inlet profile integrates to zero")
    g = np.zeros((mesh.num_nodes, 3, N))
    mag = shape[nodes][:, None] * q[None, :] / integral  # (n_inlet, N)
    g[nodes] = mag[:, None, :] * d[None, :, None]
    return g.reshape(-1)


def time_dirichlet(mesh: Mesh, inlet: int, Q0: float, a, b, period: float):
    """TimeDirichletFn for the time-stepping solver (cases.hpp:132-133): the
    ParabolicRound inlet profile of `parabolic_dirichlet` carrying
    Q(t) = Q0 (1 + sum_k a_k cos(2 pi k t / T) + b_k sin(2 pi k t / T)), and
    dQ/dt, evaluated analytically.  Returns fn(t) -> (g, gdot), node*3+i."""
    shape = parabolic_dirichlet(mesh, inlet, np.ones(1))  # unit-flow profile
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    k = np.arange(1, len(a) + 1)
    w = 2.0 * np.pi / period

    def fn(t: float):
        q = Q0 * (1.0 + float(np.sum(a * np.cos(w * k * t) + b * np.sin(w * k * t))))
        dq = Q0 * float(np.sum(w * k * (-a * np.sin(w * k * t) + b * np.cos(w * k * t))))
        return shape * q, shape * dq

    return fn


def config_problem(cfg: int, modes: int | None = None, mesh: Mesh | None = None) -> Problem:
    """BASELINE.json configs 0-3 (rho 1.06, mu 0.04, T = 1, no-slip walls,
    zero-traction outlets, parabolic pulsatile inflow).
      0/1: hex-mapped pipe, one inlet (Nm 3 / 10);
      2:   T-junction, two Dirichlet inlets carrying Q1, Q2 with seeded means
           U(15, 25) mL/s and the config-1 harmonic shape (Nm 10) — beyond
           build_case's single inlet (cases.cpp:653-658): dirichlet_g is
           supplied directly, as SURVEY.md §8(d) prescribes;
      3:   curved tapered stenosis, coronary-like inflow with 16 seeded
           harmonics (Nm 16: k = 16 is out of band and truncated); the
           BASELINE resistance outlet (R = 1e4) is not in the reference, so
           parity and timing use zero traction.
    `mesh` overrides the full-size generator (tests use small meshes)."""
    mesh = meshgen.config_mesh(cfg) if mesh is None else mesh
    M = modes if modes is not None else {0: 3, 1: 10, 2: 10, 3: 16}[cfg]
    Q0, a, b = inflow_coefficients(cfg)
    if cfg == 2:
        means = np.random.default_rng(cfg + 100).uniform(15.0, 25.0, 2)
        g = sum(parabolic_dirichlet(mesh, mesh.patch_index(name), flow_samples(qm, a, b, M, 1.0))
                for name, qm in zip(("inlet1", "inlet2"), means))
    else:
        q = flow_samples(Q0, a, b, M, 1.0)
        g = parabolic_dirichlet(mesh, mesh.patch_index("inlet"), q)
    N = 2 * M - 1
    neumann = [(k, np.zeros(N)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    return Problem(mesh, M, 1.0, 1.06, 0.04, g, neumann, 0.2)


def random_state(nn: int, N: int, seed: int, amp: float = 1.0) -> np.ndarray:
    """u, p ~ U(-amp, amp) (the random states of test_assembly.cpp:43-50),
    seeded numpy PCG64 so both sides read identical bits."""
    return np.random.default_rng(seed).uniform(-amp, amp, size=nn * 4 * N)


def random_modes_state(nn: int, modes: int, seed: int) -> np.ndarray:
    """Config 4 state: per (node, field) c_0 ~ N(0,1), c_k = (a+ib)/k^2,
    a, b ~ N(0,1), c_-k = conj(c_k); samples v_n = sum_k c_k e^{2 pi i k n/N}."""
    N = 2 * modes - 1
    rng = np.random.default_rng(seed)
    c0 = rng.standard_normal((nn * 4, 1))
    v = np.repeat(c0, N, axis=1)
    n = np.arange(N)
    for k in range(1, modes):
        ck = (rng.standard_normal((nn * 4, 1)) + 1j * rng.standard_normal((nn * 4, 1))) / k**2
        v = v + 2.0 * np.real(ck * np.exp(2j * np.pi * k * n / N)[None, :])
    return v.reshape(-1)


def initial_state(prob: Problem) -> np.ndarray:
    """Newton iterate 0: rest + Dirichlet g + outlet pressure level
    (hb_solver.cpp:119-132, assembly.cpp:415-441)."""
    mesh, N = prob.mesh, prob.N
    s = np.zeros((mesh.num_nodes, 4, N))
    g = prob.dirichlet_g.reshape(mesh.num_nodes, 3, N)
    d = mesh.dirichlet.astype(bool)
    s[d, :3, :] = g[d]
    wsum = acc = 0.0
    for pidx, h in prob.neumann:
        area = mesh.patches[pidx].area
        acc += area * (-np.mean(h))
        wsum += area
    p0 = acc / wsum if wsum > 0 else 0.0
    if p0 != 0.0:
        s[:, 3, :] = p0
    return s.reshape(-1)
