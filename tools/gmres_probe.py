"""Short GMRES run on config 1 for kernel-level profiling (ncu launch lists)."""
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_14315_b200 import cases, hbgpu  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 60
prob = cases.config_problem(1)
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
e0.record(st)
out = ctx.gmres_dev(r.data_ptr(), x.data_ptr(), hbgpu.KrylovConfig(200, iters, 1e-12))
e1.record(st)
torch.cuda.synchronize()
print("gmres", out, "ms", e0.elapsed_time(e1), "per iter", e0.elapsed_time(e1) / max(out[0], 1))
