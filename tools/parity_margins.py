"""Print the normwise relative errors of the GPU path against the restated
oracle on config 1 and a Delaunay cube (how much margin the 1e-12 bar has).
Uses HBGPU_LIB if set (variant libraries)."""
import numpy as np

from oracle import bindings as ob
from paper_2411_14315_b200 import cases, meshgen
from paper_2411_14315_b200.cases import Problem
from paper_2411_14315_b200.hbgpu import GpuContext


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run(prob, tag, tau=0):
    ctx = GpuContext(prob.mesh)
    ctx.set_basis(prob.modes, prob.period)
    ctx.set_fluid(prob.rho, prob.mu)
    ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
    ctx.set_assembly_config(tau, 0.05)
    orc = ob.Restated(prob, tau_mode=tau, pseudo_dt=0.05)
    s = cases.random_state(prob.mesh.num_nodes, prob.N, 3, 2.0)
    print(tag, "residual", rel(ctx.assemble_residual(s), orc.residual(s)),
          "tangent", rel(ctx.assemble_tangent(s), orc.tangent(s)), flush=True)


run(cases.config_problem(1), "config1")
m = meshgen.cube_delaunay(20000, seed=3)
N = 19
neu = [(k, np.full(N, 50.0)) for k, p in enumerate(m.patches) if p.kind == 1]
run(Problem(m, 10, 1.0, 1.06, 0.04, np.zeros(m.num_nodes * 3 * N), neu, 0.2), "delaunay")
