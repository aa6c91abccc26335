"""Fine-level transfers of the configs[3] hierarchy, for ncu captures and event timing:
the masked prolongation-add (level 9 -> 10) and the zeroing restriction (10 -> 9),
each after warm-up (python tools/prof_transfer.py [--level L] [--reps R])."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=10)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
L = _lib.load()
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe", seed=0, notch=True)
st = P.LinearizationState(h, 10, params, split="miehe")
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
st.set_dirichlet_nodes(dirn)
gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
gmg.setup(st)
s = torch.cuda.current_stream().cuda_stream
l = a.level
hf, hc = gmg.states[l].bind(), gmg.states[l - 1].bind()
nf, nc = gmg.states[l].n_scalar, gmg.states[l - 1].n_scalar
g = torch.Generator(device="cuda").manual_seed(l)
xc = torch.rand(3 * nc, dtype=torch.float64, device="cuda", generator=g)
yf = torch.rand(3 * nf, dtype=torch.float64, device="cuda", generator=g)
rc = torch.empty(3 * nc, dtype=torch.float64, device="cuda")
ops = {"prolong_add": lambda: L.pff_prolongate(hf, hc, xc.data_ptr(), yf.data_ptr(), 1, s),
       "prolong": lambda: L.pff_prolongate(hf, hc, xc.data_ptr(), yf.data_ptr(), 0, s),
       "restrict": lambda: L.pff_restrict(hf, hc, yf.data_ptr(), rc.data_ptr(), 1, s)}
torch.cuda.synchronize()
torch.cuda.profiler.start()   # ncu --profile-from-start off: the setup is not captured
for name, fn in ops.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(a.reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    print(f"level {l} {name}: {ev[0].elapsed_time(ev[1]) / a.reps * 1e3:.1f} us", flush=True)
