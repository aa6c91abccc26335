"""A/B of the level transfers: the current library vs a previous build
(tools/_ab/libpff_old.so, same Level layout) on the configs[3] hierarchy --
bitwise comparison and CUDA-event timing per level
(python tools/ab_transfer.py on a GPU)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import _lib  # noqa: E402

new = _lib.load()
old = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ab", "libpff_old.so"))
for L in (new, old):
    for f in ("pff_prolongate", "pff_restrict"):
        getattr(L, f).argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_void_p]
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe", seed=0, notch=True)
st = P.LinearizationState(h, 10, params, split="miehe")
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
st.set_dirichlet_nodes(dirn)
gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
gmg.setup(st)
s = torch.cuda.current_stream().cuda_stream


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps * 1e3


for l in range(10, 2, -1):
    hf, hc = gmg.states[l].bind(), gmg.states[l - 1].bind()
    nf, nc = gmg.states[l].n_scalar, gmg.states[l - 1].n_scalar
    g = torch.Generator(device="cuda").manual_seed(l)
    xc = torch.rand(3 * nc, dtype=torch.float64, device="cuda", generator=g)
    yf = torch.rand(3 * nf, dtype=torch.float64, device="cuda", generator=g)
    out = {}
    for name, lib in (("new", new), ("old", old)):
        p0 = torch.empty(3 * nf, dtype=torch.float64, device="cuda")
        p1 = yf.clone()
        r0 = torch.empty(3 * nc, dtype=torch.float64, device="cuda")
        lib.pff_prolongate(hf, hc, xc.data_ptr(), p0.data_ptr(), 0, s)
        lib.pff_prolongate(hf, hc, xc.data_ptr(), p1.data_ptr(), 1, s)
        lib.pff_restrict(hf, hc, yf.data_ptr(), r0.data_ptr(), 1, s)
        tp = timed(lambda: lib.pff_prolongate(hf, hc, xc.data_ptr(), p0.data_ptr(), 0, s))
        tr = timed(lambda: lib.pff_restrict(hf, hc, yf.data_ptr(), r0.data_ptr(), 1, s))
        tpa = timed(lambda: lib.pff_prolongate(hf, hc, xc.data_ptr(), p1.data_ptr(), 1, s))
        out[name] = (p0, p1, r0, tp, tr, tpa)
    same = [torch.equal(a, b) for a, b in zip(out["new"][:3], out["old"][:3])]
    print(f"level {l}: prolong-add {out['old'][5]:.1f} -> {out['new'][5]:.1f} us, "
          f"prolong {out['old'][3]:.1f} -> {out['new'][3]:.1f} us, "
          f"restrict {out['old'][4]:.1f} -> {out['new'][4]:.1f} us, bitwise {same}", flush=True)
