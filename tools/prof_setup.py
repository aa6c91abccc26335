"""Wall-clock breakdown of GmgPreconditioner.setup on configs[3]."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import multigrid as MG, operator as OP  # noqa: E402

split = sys.argv[1] if len(sys.argv) > 1 else "miehe"
level = 10
T = {}


def timed(name, fn):
    def wrap(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return out
    return wrap


for rep in range(2):
    T.clear()
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, level, split, seed=0, notch=True)
    st = P.LinearizationState(h, level, params, split=split)
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    timed("refresh_fine", st.refresh_cache)()
    gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    MG.op.restrict_state_to_level = timed("inject", OP.restrict_state_to_level)
    MG.op.block_diagonals = timed("diag", OP.block_diagonals)
    gmg._estimate_ranges = timed("lanczos", gmg._estimate_ranges)
    gmg.setup(st)
    timed("graph_capture", gmg.run_cycle)()
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"rep {rep}: total {tot:.3f} s; " + ", ".join(f"{k} {v:.3f}" for k, v in T.items()))
