"""Phase split of the GPU time solver on config 0 (first `steps` steps of the
500-step cycle).  python tools/time_phases.py [steps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_14315_b200 import cases, hbgpu  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
prob = cases.config_problem(0)
mesh = prob.mesh
Q0, a, b = cases.inflow_coefficients(0)
fn = cases.time_dirichlet(mesh, mesh.patch_index("inlet"), Q0, a, b, 1.0)
ctx = hbgpu.GpuContext(mesh)
ctx.set_basis(1, 1.0)
ctx.set_fluid(1.06, 0.04)
ctx.set_bcs(None, [(k, np.array([0.0])) for k, p in enumerate(mesh.patches) if p.kind == 1], 0.2)
cfg = hbgpu.TimeSolverConfig(steps_per_cycle=steps, cycles=1)
ctx.solve_time(fn, cfg, period=steps / 500.0)
L = hbgpu._lib
L.hbgpu_profile_enable.argtypes = [hbgpu._vp, hbgpu.C.c_int]
L.hbgpu_profile_read.argtypes = [hbgpu._vp, hbgpu.C.c_int, hbgpu._vp, hbgpu._vp]
L.hbgpu_profile_enable(ctx.handle, 1)
t0 = time.perf_counter()
sol = ctx.solve_time(fn, cfg, period=steps / 500.0)
wall = time.perf_counter() - t0
ms = np.zeros(13)
cnt = np.zeros(13, np.int32)
L.hbgpu_profile_read(ctx.handle, 13, ms.ctypes.data, cnt.ctypes.data)
print(f"steps {sol.total_steps} newton {sol.total_newton_iters} wall {wall * 1e3:.1f} ms "
      f"({wall * 1e3 / sol.total_steps:.2f} ms/step)")
names = ["residual", "res_hu", "res_elem", "res_final", "tangent", "matvec", "jacobi", "gmres", "mass",
         "gm_dots", "gm_arnoldi", "gm_update", "gm_matvec"]
for k, nm in enumerate(names):
    if cnt[k]:
        print(f"  {nm:12s} {ms[k]:9.2f} ms total  {1e3 * ms[k] / cnt[k]:8.1f} us x {cnt[k]}")
