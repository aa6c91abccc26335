"""GMRES iteration counts of the configs[3]/[4] Newton-step solve across mesh
levels on the device (notch phi0, seed 0, sweeps=3, rtol 1e-8), restarted
(GMRES(50), the reference's setting) and, where the basis fits, unrestarted,
plus the per-level Lanczos ranges -- the data behind the configs[4]
iteration count.

    python tools/newton_levels.py --levels 8 9 10 11 12 --split miehe \
        --unrestarted 11 > gpurun_out/newton_levels.jsonl
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402


def run(level, split, restart, max_it=1000):
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, level, split, seed=0, notch=True)
    st = P.LinearizationState(h, level, params, split=split)
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    rhs = x.copy()
    rhs[st.constrained_mask()] = 0.0
    gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    t0 = time.perf_counter()
    res = P.gmres_solve(P.JacobianOperator(st), torch.from_numpy(rhs).cuda(),
                        P.KrylovConfig(relative_tolerance=1e-8, restart=restart,
                                       max_iterations=max_it),
                        preconditioner=gmg.apply)
    torch.cuda.synchronize()
    out = {"level": level, "split": split, "restart": restart, "iterations": res.iterations,
           "converged": res.converged, "seconds": round(time.perf_counter() - t0, 3),
           "history": [float(v) for v in res.residual_history],
           "ranges": {l: [r["uu"][0], r["uu"][1], r["phiphi"][0], r["phiphi"][1]]
                      for l, r in sorted(gmg.ranges.items())}}
    del res, gmg, st
    import gc
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", type=int, nargs="+", default=[8, 9, 10, 11, 12])
    ap.add_argument("--split", default="miehe")
    ap.add_argument("--unrestarted", type=int, nargs="*", default=[8, 9, 10, 11],
                    help="levels also solved with restart 300 (basis must fit in HBM)")
    args = ap.parse_args()
    for level in args.levels:
        print(json.dumps(run(level, args.split, 50)), flush=True)
        if level in args.unrestarted:
            print(json.dumps(run(level, args.split, 300)), flush=True)


if __name__ == "__main__":
    main()
