"""GMG setup of the configs[3] hierarchy with the current library (or PFF_LIB):
every Lanczos range as an exact hex float (diff two runs for a bitwise A/B) and
the wall time of warm re-setups of one preconditioner object."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402

split = sys.argv[1] if len(sys.argv) > 1 else "miehe"
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, split, seed=0, notch=True)
st = P.LinearizationState(h, 10, params, split=split)
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
st.set_dirichlet_nodes(dirn)
st.refresh_cache()
gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
ts = []
for _ in range(6):
    torch.cuda.synchronize()
    t = time.perf_counter()
    gmg.setup(st)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t)
for l in sorted(gmg.ranges):
    for blk, (lo, hi) in sorted(gmg.ranges[l].items()):
        print(f"range {l} {blk} {float(lo).hex()} {float(hi).hex()}")
print("setup_s", " ".join(f"{t:.4f}" for t in ts[1:]), "median", f"{sorted(ts[1:])[2]:.4f}", flush=True)
