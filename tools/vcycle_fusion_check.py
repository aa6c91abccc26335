"""V-cycle with the Chebyshev start folded into the residual producers
(pff_smooth_init, pff_apply_emit) vs the separate pff_cheb_init passes: must be
bitwise identical (python tools/vcycle_fusion_check.py on a GPU)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2005_00331_b200 as P
from paper_2005_00331_b200 import multigrid as MG
for level, split in ((5, "miehe"), (8, "miehe"), (8, "none")):
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, level, split, seed=0, notch=True)
    st = P.LinearizationState(h, level, params, split=split)
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act); st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    out = {}
    for fuse in (True, False):
        MG.FUSE_INIT = fuse
        MG.EMIT_FULL = fuse
        g = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
        g.setup(st)
        out[fuse] = g.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    MG.FUSE_INIT = True
    MG.EMIT_FULL = False
    print(level, split, "bitwise" if np.array_equal(out[True], out[False]) else
          f"DIFF {np.abs(out[True]-out[False]).max()}")
