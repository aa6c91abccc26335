"""e2e (pinned host in -> device -> host out) time of apply_jacobian on configs[1]
for several pipeline chunk counts."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import operator as OP  # noqa: E402

h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe")
st = P.LinearizationState(h, 10, params, split="miehe")
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
st.set_dirichlet_nodes(dirn)
st.refresh_cache()
xh = torch.from_numpy(x).pin_memory()
xd = torch.from_numpy(x).cuda()
yd = torch.empty_like(xd)
st.apply_into(0, xd, yd)
RAMPS = {"uniform8": None, "ramp10": (1, 2, 4, 4, 4, 4, 4, 4, 2, 1),
         "ramp12": (1, 2, 3, 4, 4, 4, 4, 4, 4, 3, 2, 1), "ramp8": (1, 3, 4, 4, 4, 4, 3, 1),
         "ramp14": (1, 1, 2, 4, 4, 4, 4, 4, 4, 4, 4, 2, 1, 1)}
for K, ramp in RAMPS.items():
    OP._PIPE_CHUNKS = 8
    OP._PIPE_RAMP = ramp
    for _ in range(3):
        y = P.apply_jacobian(st, xh)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        y = P.apply_jacobian(st, xh)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 20
    assert torch.equal(y.cuda(), yd)
    print(f"{K}: {dt * 1e3:.2f} ms  {3 * st.n_scalar / dt / 1e9:.2f} GDoF/s")
