"""A/B of the two q-point cache forms of the Q2 sweep kernel (full weighted
tangent vs lean eigen-frame/strain) on the configs[1] inputs: per split and
mode the CUDA-event time per application and the relative L2 difference of
the outputs per block (python tools/sweep_forms.py --reps 200)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--level", type=int, default=10)
ap.add_argument("--splits", default="miehe,none")
ap.add_argument("--forms", default="full,lean")
a = ap.parse_args()

NAMES = {0: "FULL", 1: "UU", 2: "PHIPHI", 3: "PHIROW"}
for split in a.splits.split(","):
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, a.level, split)
    outs = {}
    for form in a.forms.split(","):
        _lib.set_option(_lib.OPT_SWEEP_CACHE, {"full": 1, "lean": 2}[form])
        st = P.LinearizationState(h, a.level, params, split=split)
        st.set_solution(U)
        st.set_phi_tilde(pt)
        st.set_phi_old(pt)
        st.set_active(act)
        st.set_dirichlet_nodes(dirn)
        st.refresh_cache()
        n = st.n_scalar
        for mode in (0, 1, 2, 3):
            nin = {0: 3 * n, 1: 2 * n, 2: n, 3: 3 * n}[mode]
            nout = {0: 3 * n, 1: 2 * n, 2: n, 3: n}[mode]
            xd = torch.from_numpy(x[:nin]).cuda()
            y = torch.empty(nout, dtype=torch.float64, device="cuda")
            for _ in range(5):
                st.apply_into(mode, xd, y)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize()
            ev[0].record()
            for _ in range(a.reps):
                st.apply_into(mode, xd, y)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1]) / a.reps
            outs.setdefault(mode, {})[form] = y.clone()
            rec = {"split": split, "form": form, "mode": NAMES[mode], "ms": round(ms, 5),
                   "gdofs_full_equiv": round(3 * n / ms / 1e6, 2) if mode == 0 else None}
            print(json.dumps(rec), flush=True)
        del st
        torch.cuda.empty_cache()
    forms = a.forms.split(",")
    if len(forms) == 2:
        for mode, d in outs.items():
            ya, yb = d[forms[0]], d[forms[1]]
            nb = ya.numel() // n
            rel = [float((ya[i * n:(i + 1) * n] - yb[i * n:(i + 1) * n]).norm() /
                         ya[i * n:(i + 1) * n].norm()) for i in range(nb)]
            print(json.dumps({"split": split, "mode": NAMES[mode], "rel_l2_full_vs_lean": rel}))
