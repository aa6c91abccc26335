"""Driver for compute-sanitizer (racecheck / synccheck / memcheck) over every
form of the Q2 sweep kernel at level 6 (64^2 cells, the smallest sweep mesh):
the four operator modes plain and fused (rhs - G src), both splits, and one
V-cycle of a level-6 hierarchy (the fused Chebyshev, emit and last forms).

    compute-sanitizer --tool racecheck python tools/sanitize_sweep.py
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import _lib  # noqa: E402

LEVEL = 6
for split in ("miehe", "none"):
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, LEVEL, split, seed=0, notch=True)
    st = P.LinearizationState(h, LEVEL, params, split=split)
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    assert st.uses_sweep_kernel()
    n = st.n_scalar
    xd = torch.from_numpy(x).cuda()
    for mode, nin, nout in ((0, 3 * n, 3 * n), (1, 2 * n, 2 * n), (2, n, n), (3, 3 * n, n)):
        y = torch.empty(nout, dtype=torch.float64, device="cuda")
        st.apply_into(mode, xd[:nin], y)
        rhs = torch.rand(nout, dtype=torch.float64, device="cuda")
        st.apply_into(mode, xd[:nin], y, rhs)
    gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    gmg.use_graph = False          # every kernel launched eagerly, one by one
    z = gmg.apply(xd)
    torch.cuda.synchronize()
    print(split, "ok", float(z.norm()))
