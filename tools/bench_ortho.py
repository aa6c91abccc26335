"""Micro-benchmark of the GMRES orthogonalisation kernels on a 1024^2 Q2-sized
basis: pff_mgs (step-by-step MGS) vs pff_mgs_lowsync, per Arnoldi column j."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_00331_b200 import _lib  # noqa: E402
from paper_2005_00331_b200._lib import call, ptr  # noqa: E402

n = 12_598_275
m = 30
L = _lib.load()
half = L.pff_reduce_scratch_len() // 2
V = torch.randn(m + 1, n, dtype=torch.float64, device="cuda")
w0 = torch.randn(n, dtype=torch.float64, device="cuda")
w = w0.clone()
part = torch.empty((2 * m + 5) * half, dtype=torch.float64, device="cuda")
h = torch.empty(m + 2, dtype=torch.float64, device="cuda")
gram = torch.zeros(m + 1, m + 1, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for j in (0, 7, 15, 29):
    for name in ("mgs", "lowsync"):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for rep in range(4):
            w.copy_(w0)
            if rep == 1:
                ev[0].record()
            if name == "mgs":
                call("pff_mgs", n, j, ptr(V), n, ptr(w), ptr(part), ptr(h), st)
            else:
                call("pff_mgs_lowsync", n, j, ptr(V), n, ptr(w), ptr(gram), m + 1, ptr(part), ptr(h), st)
        ev[1].record()
        torch.cuda.synchronize()
        # the copy w <- w0 (2 vectors) is inside the loop: subtract it
        t = ev[0].elapsed_time(ev[1]) / 3
        vecs = 4 * (j + 1) + 2 if name == "mgs" else 2 * (j + 1) + 5
        print(f"j={j:2d} {name:8s} {t*1e3:8.1f} us  ~{vecs} vector passes -> "
              f"{vecs * n * 8 / (t * 1e-3) / 1e12:.2f} TB/s (incl. the 2-vector reset copy)")
