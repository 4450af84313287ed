"""Generate the committed golden fixtures from the COMPILED REFERENCE.

Run here (where /root/reference exists and oracle/_ref/libhbref.so is built):

    python tests/golden/make_golden.py

The reference itself (oracle/_ref/libhbref.so, built by oracle/Makefile from
/root/reference/proj sources) produces every expected array; inputs are
seeded numpy PCG64 draws so the fixtures do not depend on libstdc++'s
uniform_real_distribution.  Fixtures pin the plain-C restatement
(tests/test_oracle_pin.py) on machines without the reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bindings as ob  # noqa: E402
from paper_2411_14315_b200.mesh import NEUMANN  # noqa: E402


def fixture(name, rmesh, modes, period, tau_mode, pseudo_dt, seed):
    mesh = rmesh.to_mesh()
    N = 2 * modes - 1
    rng = np.random.default_rng(seed)
    neu = [(k, rng.uniform(-1, 1, N) * 100 + 5) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    g = rng.uniform(-1, 1, mesh.num_nodes * 3 * N)
    state = rng.uniform(-1, 1, mesh.num_nodes * 4 * N)
    y = rng.uniform(-1, 1, mesh.num_nodes * 4 * N)
    ctx = ob.RefCtx(rmesh, modes, period, 1.06, 0.04)
    ctx.set_bcs(g, neu, 0.2)
    ctx.set_cfg(tau_mode, pseudo_dt)
    r = ctx.residual(state, 1)
    p = ctx.tangent(state)
    m = ctx.mass()
    mv = ctx.matvec(y, 1)
    inv, deg = ctx.jacobi()
    rp, ci = rmesh.pattern()
    gm = ctx.gmres(mv, inv, restart=40, max_iters=400, tol=1e-9)
    out = dict(
        xyz=mesh.xyz, conn=mesh.conn, dirichlet=mesh.dirichlet,
        patch_names=np.array([pp.name for pp in mesh.patches]),
        patch_kinds=np.array([pp.kind for pp in mesh.patches], np.int32),
        patch_nfacets=np.array([len(pp.facets) for pp in mesh.patches], np.int32),
        facets=np.concatenate([pp.facets for pp in mesh.patches]),
        normals=np.concatenate([pp.normals for pp in mesh.patches]),
        areas=np.concatenate([pp.areas for pp in mesh.patches]),
        geometry=rmesh.geometry(), modes=modes, period=period, tau_mode=tau_mode,
        pseudo_dt=pseudo_dt if np.isfinite(pseudo_dt) else 0.0,
        neumann_patch=np.array([k for k, _ in neu], np.int32),
        neumann_h=np.array([h for _, h in neu]), dirichlet_g=g, state=state, y=y,
        residual=r, pvals=p, mass=m, matvec=mv, inv_diag=inv, degenerate=deg,
        row_ptr=rp, col_idx=ci, H=ob.ref_h_dense(modes, period),
        gmres_x=gm["x"], gmres_iters=gm["iterations"], gmres_relres=gm["relative_residual"],
        oracle_residual=ctx.oracle_residual(state),
    )
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, mesh.num_nodes, mesh.num_elements, "nnz", len(ci), "gmres", gm["iterations"])


def main():
    fixture("tube_m3_qp", ob.RefMesh.tube(0.5, 1.0, 0.34), 3, 0.8, 0, 0.3, 1)
    fixture("tube_m4_mean", ob.RefMesh.tube(0.5, 1.0, 0.34), 4, 1.0, 1, float("inf"), 2)
    fixture("tube_m1_steady", ob.RefMesh.tube(0.5, 1.5, 0.25), 1, 1.0, 0, 0.05, 3)
    fixture("bifurcation_m3", ob.RefMesh.bifurcation(0.4, 0.4, 0.8, 0.8, 0.2), 3, 1.0, 0, 0.1, 4)
    # FFTW-path pin: SpectralOperators::apply_many vs the dense H (test_spectral.cpp:104-151)
    rng = np.random.default_rng(9)
    spec = {}
    for M in (1, 2, 3, 4, 7, 13):
        N = 2 * M - 1
        v = rng.uniform(-1, 1, 5 * N)
        spec[f"H_{M}"] = ob.ref_h_dense(M, 0.7)
        spec[f"Hora_{M}"] = ob.ref_oracle_h_dense(M, 0.7)
        spec[f"v_{M}"] = v
        spec[f"Hv_{M}"] = ob.ref_apply_h(M, 0.7, v)
    np.savez_compressed(os.path.join(HERE, "spectral.npz"), **spec)
    print("spectral ok")


if __name__ == "__main__":
    main()
