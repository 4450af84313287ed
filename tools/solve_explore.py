"""Explore pseudo-time steps for the converged solves of BASELINE configs 1-3
 on the GPU.  Tooling, not product: prints one JSON line
per (config, CFL) with the Newton log.

  python tools/solve_explore.py --configs 1,2,3 --cfl 1,3,10 --max-newton 40
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from bench import auto_pseudo_dt  # noqa: E402
from paper_2411_14315_b200 import cases, hbgpu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--cfl", default="1,3,10")
    ap.add_argument("--max-newton", type=int, default=40)
    ap.add_argument("--orders", type=float, default=3.0)
    ap.add_argument("--resistance", action="store_true", help="config 3 with R = 1e4 outlets")
    ap.add_argument("--restart", type=int, default=200)
    ap.add_argument("--max-iters", type=int, default=1000)
    ap.add_argument("--tol", type=float, default=0.03)
    args = ap.parse_args()
    for cfg in [int(c) for c in args.configs.split(",")]:
        t0 = time.time()
        prob = cases.config_problem(cfg)
        t_mesh = time.time() - t0
        dt0 = auto_pseudo_dt(prob)
        for cfl in [float(c) for c in args.cfl.split(",")]:
            ctx = hbgpu.GpuContext(prob.mesh)
            ctx.set_basis(prob.modes, prob.period)
            ctx.set_fluid(prob.rho, prob.mu)
            ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
            if cfg == 3 and args.resistance:
                ctx.set_resistance({k: 1e4 for k, _ in prob.neumann})
            sc = hbgpu.SolverConfig(pseudo_dt=dt0 * cfl, newton_tol_orders=args.orders,
                                    max_newton_iters=args.max_newton,
                                    krylov=hbgpu.KrylovConfig(args.restart, args.max_iters, args.tol))
            rec = {"config": cfg, "cfl": cfl, "pseudo_dt": dt0 * cfl, "elements": prob.mesh.num_elements,
                   "N": prob.N, "mesh_s": t_mesh}
            try:
                sol = ctx.solve_harmonic(sc)
                rec.update(converged=sol.log.converged, seconds=sol.total_seconds,
                           newton=int(len(sol.log.iters)), gmres=int(sol.log.linear_iters.sum()),
                           rel=[float(x) for x in sol.log.res_rel], lin=[int(x) for x in sol.log.linear_iters],
                           assembly_s=sol.assembly_seconds, linear_s=sol.linear_seconds)
            except Exception as exc:  # divergence / stagnation
                rec.update(error=f"{type(exc).__name__}: {exc}",
                           log=getattr(exc, "partial_log_csv", "")[-2000:])
            print(json.dumps(rec), flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
