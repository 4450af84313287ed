"""Short GMRES run on config 1 (or argv[2]) for kernel-level profiling (ncu launch lists)."""
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_14315_b200 import cases, hbgpu  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 60
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
prob = cases.config_problem(cfg)
ctx = hbgpu.GpuContext(prob.mesh)
ctx.set_basis(prob.modes, prob.period)
ctx.set_fluid(prob.rho, prob.mu)
ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
ctx.set_assembly_config(0, 0.0027)
s0 = torch.from_numpy(cases.initial_state(prob)).cuda()
r = torch.empty_like(s0)
x = torch.empty_like(s0)
ctx.assemble_residual_dev(s0.data_ptr(), r.data_ptr())
ctx.assemble_tangent_dev(s0.data_ptr())
ctx.jacobi_dev()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.ExternalStream(ctx.stream)
out = ctx.gmres_dev(r.data_ptr(), x.data_ptr(), hbgpu.KrylovConfig(200, iters, 1e-12))  # warm-up
torch.cuda.synchronize()
e0.record(st)
out = ctx.gmres_dev(r.data_ptr(), x.data_ptr(), hbgpu.KrylovConfig(200, iters, 1e-12))
e1.record(st)
torch.cuda.synchronize()
it = max(out[0], 1)
print("gmres", out, "ms", e0.elapsed_time(e1), "per iter", e0.elapsed_time(e1) / it)
# per-phase device time of the same solve (CUDA events around each launch group)
L = hbgpu._lib
L.hbgpu_profile_enable.argtypes = [hbgpu._vp, hbgpu.C.c_int]
L.hbgpu_profile_read.argtypes = [hbgpu._vp, hbgpu.C.c_int, hbgpu._vp, hbgpu._vp]
L.hbgpu_profile_enable(ctx.handle, 1)
ctx.gmres_dev(r.data_ptr(), x.data_ptr(), hbgpu.KrylovConfig(200, iters, 1e-12))
ms = np.zeros(13)
cnt = np.zeros(13, np.int32)
L.hbgpu_profile_read(ctx.handle, 13, ms.ctypes.data, cnt.ctypes.data)
L.hbgpu_profile_enable(ctx.handle, 0)
for k, name in [(12, "matvec"), (9, "dots+reduce"), (10, "arnoldi"), (11, "update+normalize")]:
    print(f"  {name:18s} {1e3 * ms[k] / max(cnt[k], 1):8.2f} us x {cnt[k]}")
