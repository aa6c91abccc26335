"""Small driver for ncu: build the configs[1] state and apply the operator a
few times (python tools/prof_apply.py --split miehe --mode 0 --reps 3)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--split", default="miehe")
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--level", type=int, default=10)
ap.add_argument("--generic", type=int, default=0)
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--degree", type=int, default=2)
ap.add_argument("--fused", type=int, default=0, help="fused residual form dst = rhs - G src")
a = ap.parse_args()
_lib.set_option(_lib.OPT_GENERIC_APPLY, a.generic)
_lib.set_option(_lib.OPT_SWEEP_ROWS, a.rows)
h, params, U, pt, act, dirn, x = bench.baseline_inputs(a.degree, a.level, a.split)
st = P.LinearizationState(h, a.level, params, split=a.split)
st.set_solution(U)
st.set_phi_tilde(pt)
st.set_phi_old(pt)
st.set_active(act)
st.set_dirichlet_nodes(dirn)
st.refresh_cache()
n = st.n_scalar
nin = {0: 3 * n, 1: 2 * n, 2: n, 3: 3 * n}[a.mode]
nout = {0: 3 * n, 1: 2 * n, 2: n, 3: n}[a.mode]
xd = torch.from_numpy(x[:nin]).cuda()
y = torch.empty(nout, dtype=torch.float64, device="cuda")
rhs = torch.rand(nout, dtype=torch.float64, device="cuda") if a.fused else None
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(a.reps):
    st.apply_into(a.mode, xd, y, rhs)
torch.cuda.synchronize()
ev[0].record()
for i in range(a.reps):
    st.apply_into(a.mode, xd, y, rhs)
ev[1].record()
torch.cuda.synchronize()
print(f"mode {a.mode} split {a.split}: {ev[0].elapsed_time(ev[1]) / a.reps:.4f} ms/apply")
