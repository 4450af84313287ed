"""GPU solve_time vs the compiled reference's on a reference tube: errors and
wall times.  python tools/time_probe.py [h] [steps] [cycles]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bindings as ob  # noqa: E402
from paper_2411_14315_b200 import cases  # noqa: E402
from paper_2411_14315_b200.hbgpu import GpuContext, KrylovConfig, TimeSolverConfig  # noqa: E402
from paper_2411_14315_b200.mesh import NEUMANN  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "0.15"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cycles = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if arg == "cfg0":  # BASELINE config 0 pipe, its inflow, dt of the 500-step cycle
    prob = cases.config_problem(0)
    mesh = prob.mesh
    rm = ob.RefMesh.from_mesh(mesh)
    Q0, a, b = cases.inflow_coefficients(0)
    fn = cases.time_dirichlet(mesh, mesh.patch_index("inlet"), Q0, a, b, 1.0)
    T = steps / 500.0
    neu = [(k, np.array([0.0])) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
else:
    T = 0.5
    rm = ob.RefMesh.tube(0.3, 0.6, float(arg))
    mesh = rm.to_mesh()
    fn = cases.time_dirichlet(mesh, mesh.patch_index("inlet"), 2.0, [0.2, -0.1], [0.1, 0.05], T)
    neu = [(k, np.array([-20.0])) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
for orders, tol, mx in ((10.0, 1e-10, 12), (3.0, 0.03, 8)):
    ref = ob.RefCtx(rm, 1, T)
    ref.set_bcs(None, neu, 0.2)
    t0 = time.perf_counter()
    r = ref.solve_time(fn, T, steps=steps, cycles=cycles, orders=orders, max_newton=mx, tol=tol)
    tr = time.perf_counter() - t0
    ctx = GpuContext(mesh)
    ctx.set_basis(1, T)
    ctx.set_fluid(1.06, 0.04)
    ctx.set_bcs(None, neu, 0.2)
    cfg = TimeSolverConfig(steps, cycles, 0.2, orders, mx, KrylovConfig(200, 1000, tol))
    ctx.solve_time(fn, cfg)  # warm-up
    t0 = time.perf_counter()
    g = ctx.solve_time(fn, cfg)
    tg = time.perf_counter() - t0
    eu = max(rel(g.u[j], r["u"][j]) for j in range(g.u.shape[0]))
    ep = max(rel(g.p[j], r["p"][j]) for j in range(g.p.shape[0]))
    print(f"nodes {mesh.num_nodes} elems {mesh.num_elements} steps {steps}x{cycles} orders {orders}: "
          f"max rel u {eu:.2e} p {ep:.2e}; newton gpu {g.total_newton_iters} ref {r['total_newton_iters']}; "
          f"cycle_change {g.cycle_change:.6e} / {r['cycle_change']:.6e}; gpu {tg:.3f}s ref {tr:.3f}s")
