"""Steady-state phase breakdown of GmgPreconditioner.setup on configs[3] (the
second setup in the process), wall clock with device synchronisation."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import multigrid as MG, operator as OP  # noqa: E402

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


h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe", seed=0, notch=True)
MG.op.restrict_state_to_level = timed("inject+coarse refresh", OP.restrict_state_to_level)
MG.op.block_diagonals = timed("diagonals", OP.block_diagonals)
MG.GmgPreconditioner._estimate_ranges_batched = timed(
    "lanczos", MG.GmgPreconditioner._estimate_ranges_batched)
MG.GmgPreconditioner._build_dense_coarse = timed(
    "dense coarse", MG.GmgPreconditioner._build_dense_coarse)
EMPTY = "--empty-cache" in sys.argv   # bench.py's pattern: release the cache between solves
for rep in range(3):
    T.clear()
    if EMPTY:
        import gc
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    st = P.LinearizationState(h, 10, params, split="miehe")
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    timed("refresh fine", st.refresh_cache)()
    gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    timed("setup total", gmg.setup)(st)
    timed("graph capture", gmg.run_cycle)()
    tot = time.perf_counter() - t0
    print(f"rep {rep}: total {tot * 1e3:.1f} ms; " + ", ".join(f"{k} {v * 1e3:.1f}" for k, v in T.items()))
