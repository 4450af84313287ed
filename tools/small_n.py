"""Operator timing at a given Nm on a Delaunay cube (small-N investigation).
python tools/small_n.py [points] [Nm] [reps]"""
import sys
import time

import numpy as np
import torch

from paper_2411_14315_b200 import cases, hbgpu, meshgen

pts = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
mesh = meshgen.cube_delaunay(pts, seed=4)
N = 2 * M - 1
ctx = hbgpu.GpuContext(mesh)
ctx.set_basis(M, 1.0)
ctx.set_fluid(1.06, 0.04)
ctx.set_bcs(None, [(k, np.zeros(N)) for k, p in enumerate(mesh.patches) if p.kind == 1], 0.2)
ctx.set_assembly_config(0, 0.01)
s = torch.from_numpy(cases.random_modes_state(mesh.num_nodes, M, 1)).cuda()
r = torch.empty_like(s)
for _ in range(reps):
    ctx.assemble_residual_dev(s.data_ptr(), r.data_ptr())
    ctx.assemble_tangent_dev(s.data_ptr())
ctx.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    ctx.assemble_tangent_dev(s.data_ptr())
ctx.synchronize()
print("elements", mesh.num_elements, "N", N, "tangent ms", (time.perf_counter() - t0) / reps * 1e3)
