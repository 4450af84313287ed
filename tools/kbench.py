"""Element-kernel A/B timing (tooling, not product): residual and tangent of
one state, each alone (CUDA events on the library stream, L2 flushed before
each launch, median of 5), for configs 1 (N=19) and 4 (Nm=24, N=47) or a
reduced config 4, for one or more builds of libhbgpu.so.

  python tools/kbench.py --libs paper_2411_14315_b200/libhbgpu.so,paper_2411_14315_b200/variants/libhbgpu_x.so
Each library runs in its own process (HBGPU_LIB is read at import); meshes
are pickled to /tmp once per call.
"""
import argparse
import json
import os
import pickle
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CANON_RES, CANON_TAN = 1198, 1532


def make_problems(which, points):
    import numpy as np

    from paper_2411_14315_b200 import cases, meshgen
    from paper_2411_14315_b200.mesh import NEUMANN

    out = {}
    for w in which.split(","):
        path = f"/tmp/kbench_{w}_{points}.pkl"
        if os.path.exists(path):
            continue
        if w == "c1":
            prob = cases.config_problem(1)
            st = cases.random_state(prob.mesh.num_nodes, prob.N, 1001)
        else:
            M = int(w[3:]) if w.startswith("c4m") else 24
            mesh = meshgen.cube_delaunay(points, seed=4)
            N = 2 * M - 1
            neu = [(k, np.zeros(N)) for k, p in enumerate(mesh.patches) if p.kind == NEUMANN]
            prob = cases.Problem(mesh, M, 1.0, 1.06, 0.04, np.zeros(mesh.num_nodes * 3 * N), neu, 0.2)
            st = cases.random_modes_state(mesh.num_nodes, M, 1000 + M)
        with open(path, "wb") as f:
            pickle.dump((prob, st), f)
        out[w] = path
    return out


def run_one(which, points, reps):
    import numpy as np
    import torch

    from paper_2411_14315_b200 import hbgpu

    L = hbgpu._lib
    L.hbgpu_profile_enable.argtypes = [hbgpu._vp, hbgpu.C.c_int]
    L.hbgpu_profile_read.argtypes = [hbgpu._vp, hbgpu.C.c_int, hbgpu._vp, hbgpu._vp]
    res = {"lib": hbgpu.LIB_PATH}
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for w in which.split(","):
        with open(f"/tmp/kbench_{w}_{points}.pkl", "rb") as f:
            prob, st = pickle.load(f)
        ctx = hbgpu.GpuContext(prob.mesh)
        ctx.set_basis(prob.modes, prob.period)
        ctx.set_fluid(prob.rho, prob.mu)
        ctx.set_bcs(prob.dirichlet_g, prob.neumann, prob.backflow_beta)
        ctx.set_assembly_config(0, 0.01)
        stream = torch.cuda.ExternalStream(ctx.stream)
        d_s = torch.from_numpy(st).cuda()
        d_r = torch.empty_like(d_s)
        for _ in range(2):
            ctx.assemble_residual_dev(d_s.data_ptr(), d_r.data_ptr())
            ctx.assemble_tangent_dev(d_s.data_ptr())
        torch.cuda.synchronize()

        def timed(fn):
            ts = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    flush.fill_(1.0)
                    a.record(stream)
                    fn()
                    b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            return float(np.median(ts))

        L.hbgpu_profile_enable(ctx.handle, 1)
        t_res = timed(lambda: ctx.assemble_residual_dev(d_s.data_ptr(), d_r.data_ptr()))
        ms = np.zeros(14)
        cnt = np.zeros(14, np.int32)
        L.hbgpu_profile_read(ctx.handle, 14, ms.ctypes.data, cnt.ctypes.data)
        L.hbgpu_profile_enable(ctx.handle, 0)
        t_tan = timed(lambda: ctx.assemble_tangent_dev(d_s.data_ptr()))
        t_both = timed(lambda: ctx.assemble_dev(d_s.data_ptr(), d_r.data_ptr()))
        y = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, st.size)).cuda()
        o = torch.empty_like(y)
        ctx.assemble_mass()

        def mv10():
            for _ in range(10):
                ctx.matvec_dev(y.data_ptr(), o.data_ptr())

        t_mv = timed(mv10) / 10
        nnz = ctx.nnz
        mvb = 64 * prob.N * nnz + 12 * nnz + 4 * (prob.mesh.num_nodes + 1) + 64 * prob.N * prob.mesh.num_nodes + prob.mesh.num_nodes
        del y, o
        ne, N = prob.mesh.num_elements, prob.N
        res[w] = {"elements": ne, "N": N, "residual_ms": t_res, "tangent_ms": t_tan, "step_ms": t_both,
                  "res_elem_ms": float(ms[2] / max(cnt[2], 1)), "res_hu_ms": float(ms[1] / max(cnt[1], 1)),
                  "res_final_ms": float(ms[3] / max(cnt[3], 1)), "tau_ms": float(ms[13] / max(cnt[13], 1)),
                  "res_tflops": CANON_RES * ne * N / (t_res * 1e-3) / 1e12,
                  "tan_tflops": CANON_TAN * ne * N / (t_tan * 1e-3) / 1e12,
                  "matvec_ms": t_mv, "matvec_gbs": mvb / (t_mv * 1e-3) / 1e9}
        # parity of this build against the first library's outputs is checked by the caller
        r = d_r.cpu().numpy()
        np.save(f"/tmp/kbench_out_{w}_{os.path.basename(hbgpu.LIB_PATH)}_r.npy", r[: 4 * N * 2000])
        # a spread of P block rows (first, last and a stride through the mesh); compared with the
        # first library's by the caller
        nn = prob.mesh.num_nodes
        rows = np.unique(np.concatenate([np.arange(0, nn, max(1, nn // 1500)), np.arange(nn - 50, nn)])).astype(np.int32)
        ctx.assemble_tangent_dev(d_s.data_ptr())
        torch.cuda.synchronize()
        pr = ctx.pvals_rows(rows)
        np.save(f"/tmp/kbench_out_{w}_{os.path.basename(hbgpu.LIB_PATH)}_p.npy", pr)
        ctx.close()
        del d_s, d_r
        torch.cuda.empty_cache()
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", default=os.path.join(ROOT, "paper_2411_14315_b200", "libhbgpu.so"))
    ap.add_argument("--which", default="c1,c4")
    ap.add_argument("--points", type=int, default=700_000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    if args.child:
        run_one(args.which, args.points, args.reps)
        return
    make_problems(args.which, args.points)
    first = None
    for lib in args.libs.split(","):
        env = dict(os.environ, HBGPU_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, __file__, "--child", "--which", args.which, "--points",
                              str(args.points), "--reps", str(args.reps)], env=env, capture_output=True,
                             text=True)
        print(out.stdout.strip() or out.stderr[-2000:], flush=True)
        import numpy as np
        base = os.path.basename(os.path.abspath(lib))
        first = first or base
        for w in args.which.split(","):
            for kind in ("r", "p"):
                try:
                    x = np.load(f"/tmp/kbench_out_{w}_{base}_{kind}.npy")
                    y = np.load(f"/tmp/kbench_out_{w}_{first}_{kind}.npy")
                    print(f"  parity {w} {kind}: rel diff vs {first} = {np.linalg.norm(x - y) / np.linalg.norm(y):.2e}", flush=True)
                except Exception as e:  # noqa: BLE001
                    print(f"  parity {w} {kind}: {e}", flush=True)


if __name__ == "__main__":
    main()
