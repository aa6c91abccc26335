"""Lanczos phase of the GMG setup (configs[3]): wall time vs summed device
time of its kernels, and the device time per kernel family."""
import os
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import multigrid as MG  # noqa: E402

h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe", seed=0, notch=True)
orig = MG.GmgPreconditioner._estimate_ranges_batched
box = {}


def wrapped(self, levels):
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    if box.get("profile"):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            t0 = time.perf_counter()
            out = orig(self, levels)
            torch.cuda.synchronize()
            box["wall"] = time.perf_counter() - t0
        box["prof"] = prof
        return out
    return orig(self, levels)


MG.GmgPreconditioner._estimate_ranges_batched = wrapped
for rep in range(3):
    box["profile"] = rep == 2
    st = P.LinearizationState(h, 10, params, split="miehe")
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    g = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    g.setup(st)
ev = [e for e in box["prof"].events() if e.device_type == torch.autograd.DeviceType.CUDA]
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    nm = e.name.replace("pff::(anonymous namespace)::", "").replace("void ", "").split("(")[0][:50]
    agg[nm][0] += 1
    agg[nm][1] += e.device_time_total
tot = sum(v[1] for v in agg.values())
print(f"lanczos wall {box['wall'] * 1e3:.1f} ms (profiled), device sum {tot / 1e3:.1f} ms, {len(ev)} kernels")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"  {t / 1e3:8.2f} ms x{c:5d}  {k}")
ev.sort(key=lambda e: e.time_range.start)
span = (ev[-1].time_range.end - ev[0].time_range.start) / 1e3
print(f"device span {span:.1f} ms")
