"""Load the committed golden fixtures (tests/golden/*.npz, made from the
compiled reference by tests/golden/make_golden.py) as Problems."""
import os

import numpy as np

from paper_2411_14315_b200.cases import Problem
from paper_2411_14315_b200.mesh import Mesh, Patch

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["tube_m3_qp", "tube_m4_mean", "tube_m1_steady", "bifurcation_m3"]


def load(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    patches, off = [], 0
    for nm, kind, nf in zip(d["patch_names"], d["patch_kinds"], d["patch_nfacets"]):
        nf = int(nf)
        patches.append(Patch(str(nm), int(kind), d["facets"][off:off + nf].astype(np.int32),
                             d["normals"][off:off + nf], d["areas"][off:off + nf]))
        off += nf
    mesh = Mesh(d["xyz"], d["conn"].astype(np.int32), patches, d["dirichlet"].astype(np.uint8))
    modes = int(d["modes"])
    neu = [(int(k), h) for k, h in zip(d["neumann_patch"], d["neumann_h"])]
    prob = Problem(mesh, modes, float(d["period"]), 1.06, 0.04, d["dirichlet_g"], neu, 0.2)
    pdt = float(d["pseudo_dt"])
    d["pseudo_dt_eff"] = pdt if pdt > 0 else float("inf")
    return prob, d
