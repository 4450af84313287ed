"""L-matvec timing on a Delaunay cube (BASELINE config 4) or the config-1 pipe.
python tools/mv_probe.py [points|pipe] [Nm] [reps]
Prints ms per matvec and GB/s of compulsory bytes; HBGPU_MV_VARIANT selects a
kernel variant inside libhbgpu (tooling only)."""
import os
import sys
import time

import numpy as np
import torch

from paper_2411_14315_b200 import cases, hbgpu, meshgen

arg = sys.argv[1] if len(sys.argv) > 1 else "200000"
Ms = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "10").split(",")]
variants = (sys.argv[3] if len(sys.argv) > 3 else "0").split(",")
reps = 100
t0 = time.perf_counter()
mesh = (meshgen.hex_cylinder(0.3, 6.0, 20, 20, 120) if arg == "pipe" else
        meshgen.hex_cylinder(0.3, 6.0, 10, 10, 60) if arg == "pipe0" else
        meshgen.config_mesh(int(arg[3:])) if arg.startswith("cfg") else meshgen.cube_delaunay(int(arg), seed=4))
tm = time.perf_counter() - t0


def run(M, var):
    os.environ["HBGPU_MV_VARIANT"] = var
    N = 2 * M - 1
    ctx = hbgpu.GpuContext(mesh)
    ctx.set_basis(M, 1.0)
    ctx.set_fluid(1.06, 0.04)
    ctx.set_bcs(None, [(k, np.zeros(N)) for k, p in enumerate(mesh.patches) if p.kind == 1], 0.2)
    ctx.set_assembly_config(0, 0.01)
    s = torch.from_numpy(cases.random_modes_state(mesh.num_nodes, M, 1)).cuda()
    y = torch.from_numpy(cases.random_modes_state(mesh.num_nodes, M, 2)).cuda()
    o = torch.empty_like(y)
    ctx.assemble_tangent_dev(s.data_ptr())
    ctx.matvec_dev(y.data_ptr(), o.data_ptr())
    ctx.synchronize()
    B = ctx.nnz
    V = mesh.num_nodes
    byt = 64 * N * B + 12 * B + 4 * (V + 1) + 64 * N * V + V
    st = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    res = []
    for trial in range(3):
        flush.fill_(trial)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(reps):
                ctx.matvec_dev(y.data_ptr(), o.data_ptr())
            e1.record(st)
        e1.synchronize()
        res.append(e0.elapsed_time(e1) / reps)
    ms = min(res)
    print(f"var {var} mesh {arg} ({tm:.1f}s) V {V} E {mesh.num_elements} B {B} N {N}: matvec {ms:.4f} ms "
          f"{byt / ms / 1e6:.0f} GB/s  checksum {float(o.double().abs().sum()):.12e}")
    ctx.close()


for M in Ms:
    for var in variants:
        run(M, var)
