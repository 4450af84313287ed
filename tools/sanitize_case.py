"""Small case for compute-sanitizer (racecheck / synccheck / memcheck): every
hot-path kernel on tiny meshes — the residual chunk pipeline (T = 1, 2, 4
sample tiles), the tangent row pipeline (sample pairs at N = 5, single
samples at N = 47, several CTA widths), the tiled row-kernel fallback, the
nodal H pass, the L-matvec kernels, Jacobi and the device-resident GMRES
cycle.  Tooling, not product.  Exit code 0 iff the results still match the
restatement (so a sanitizer-perturbed schedule that changed results shows up).

  compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import bindings as ob  # noqa: E402
from paper_2411_14315_b200 import cases, hbgpu, meshgen  # noqa: E402
from paper_2411_14315_b200.mesh import NEUMANN  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run(mesh, modes, env):
    os.environ.update(env)
    N = 2 * modes - 1
    neu = [(k, np.full(N, 10.0)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
    prob = cases.Problem(mesh, modes, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 3 * N), neu, 0.2)
    ctx = hbgpu.GpuContext(mesh)
    ctx.set_basis(modes, 1.0)
    ctx.set_fluid(1.06, 0.04)
    ctx.set_bcs(prob.dirichlet_g, prob.neumann, 0.2)
    ctx.set_assembly_config(0, 0.05)
    orc = ob.Restated(prob, tau_mode=0, pseudo_dt=0.05)
    s = cases.random_modes_state(mesh.num_nodes, modes, 3)
    errs = [rel(ctx.assemble_residual(s), orc.residual(s))]
    p = ctx.assemble_tangent(s)
    errs.append(rel(p, orc.tangent(s)))
    y = cases.random_state(mesh.num_nodes, N, 4)
    errs.append(rel(ctx.matvec(y), orc.matvec(p, orc.mass(), y)))
    ctx.jacobi()
    res = ctx.gmres(y, hbgpu.KrylovConfig(restart=20, max_iters=40, tolerance=1e-8))
    for k in env:
        os.environ.pop(k, None)
    return errs, res.iterations


def main():
    cube = meshgen.cube_delaunay(600, seed=5)
    tube = meshgen.hex_cylinder(0.3, 1.0, 3, 3, 4)
    worst = 0.0
    for mesh, modes, env in [
        (tube, 3, {}),                                  # pairs, residual tile 4
        (tube, 3, {"HBGPU_RES_TILE": "1"}),
        (tube, 3, {"HBGPU_TANGENT_KERNEL": "rows"}),   # tiled row-kernel fallback
        (cube, 24, {}),                                 # N = 47, compile-time-N tangent
        (cube, 24, {"HBGPU_TAN_WIDTH": "128", "HBGPU_RES_TILE": "2"}),
        (cube, 1, {"HBGPU_MV_LANES": "4"}),
    ]:
        errs, its = run(mesh, modes, env)
        worst = max(worst, max(errs))
        print(f"N={2 * modes - 1} env={env} errors={['%.1e' % e for e in errs]} gmres_iters={its}", flush=True)
    print(f"worst relative error {worst:.2e}")
    sys.exit(0 if worst < 1e-12 else 1)


if __name__ == "__main__":
    main()
