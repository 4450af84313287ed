"""Converged-solve exploration on config 0 (pseudo-dt scale, GMRES tolerance).
python tools/solve_exp.py [cfg]"""
import sys
import time

import numpy as np

import bench
from paper_2411_14315_b200 import cases, hbgpu

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for scale, gtol in ((3.0, 0.03), (10.0, 0.03), (float("inf"), 0.03), (3.0, 0.01), (10.0, 0.01)):
    prob = cases.config_problem(cfg_id)
    ctx = hbgpu.GpuContext(prob.mesh)
    ctx.set_basis(prob.modes, prob.period)
    ctx.set_fluid(prob.rho, prob.mu)
    ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
    cfg = hbgpu.SolverConfig()
    cfg.pseudo_dt = bench.auto_pseudo_dt(prob) * scale
    cfg.krylov.tolerance = gtol
    cfg.max_newton_iters = 80
    try:
        sol = ctx.solve_harmonic(cfg)
        print(f"dt x{scale} gmres {gtol}: converged {sol.log.converged} newton {len(sol.log.iters)} "
              f"gmres {int(sol.log.linear_iters.sum())} rel {sol.log.res_rel[-1]:.2e} s {sol.total_seconds:.3f}", flush=True)
    except Exception as e:
        print(f"dt x{scale} gmres {gtol}: {type(e).__name__} {e}", flush=True)
