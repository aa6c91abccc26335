"""Per-level cost of the V-cycle on one GPU, for the scaling model
(tools/scaling_model.py): the graph-captured V-cycle time T(L) of hierarchies
with finest level L = 4..Lmax (configs[3]/[4] notch inputs), the increment
T(L) - T(L-1) being level L's own cost; split into a floor (the median
increment of levels 4-6, where the size-proportional part is negligible) and a
proportional part.  Then one configs[Lmax] GMRES solve for the iteration
count, the operator time and the orthogonalisation share per iteration.

    python tools/prof_vcycle_levels.py 12 > profiles/r02/vcycle_levels_l12.json
"""

import gc
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import _lib  # noqa: E402


def state(level):
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, level, "miehe", seed=0, notch=True)
    st = P.LinearizationState(h, level, params, split="miehe")
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    return h, st, x


def timed(fn, reps):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def free():
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def main():
    lmax = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    cyc = {}
    for L in range(3, lmax + 1):
        h, st, x = state(L)
        gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
        gmg.setup(st)
        r, _ = gmg.io_buffers()
        r.copy_(torch.from_numpy(x).cuda())
        cyc[L] = timed(gmg.run_cycle, 20 if L < 11 else 5)
        if L == lmax:
            n = st.n_scalar
            xd = torch.from_numpy(x).cuda()
            yd = torch.empty_like(xd)
            t_op = timed(lambda: st.apply_into(_lib.MODE_FULL, xd, yd), 10)
            rhs = x.copy()
            rhs[st.constrained_mask()] = 0.0
            rd = torch.from_numpy(rhs).cuda()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = P.gmres_solve(P.JacobianOperator(st), rd,
                                P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                                preconditioner=gmg.apply)
            e1.record()
            torch.cuda.synchronize()
            t_gm = e0.elapsed_time(e1) * 1e-3
            its = res.iterations
            del res, rd, xd, yd
        del gmg, st
        free()
    inc = {L: cyc[L] - cyc[L - 1] for L in range(4, lmax + 1)}
    floor = float(np.median([inc[L] for L in (4, 5, 6)]))
    levels = [{"level": 3, "floor_s": cyc[3], "prop_s": 0.0, "vcycle_total_s": cyc[3]}]
    for L in range(4, lmax + 1):
        levels.append({"level": L, "floor_s": min(floor, inc[L]), "prop_s": max(inc[L] - floor, 0.0),
                       "vcycle_total_s": cyc[L]})
    ortho = t_gm / its - cyc[lmax] - t_op
    print(json.dumps({"finest": lmax, "iterations": its, "gmres_device_s": t_gm,
                      "operator_s": t_op, "ortho_s": max(ortho, 0.0), "levels": levels,
                      "how": "tools/prof_vcycle_levels.py: graph V-cycle time T(L) per finest "
                             "level L, level cost = T(L) - T(L-1), floor = median of levels 4-6"}))


if __name__ == "__main__":
    main()
