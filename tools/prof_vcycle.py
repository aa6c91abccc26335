"""Per-launch device times of ONE V-cycle (configs[3], graph off) in launch
order, aggregated per (level, kernel): where a V-cycle's time goes by level."""
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 10
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, level, "miehe", seed=0, notch=True)
st = P.LinearizationState(h, level, params, split="miehe")
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
st.set_dirichlet_nodes(dirn)
gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
gmg.setup(st)
gmg.use_graph = False
r, z = gmg.io_buffers()
r.copy_(torch.from_numpy(x).cuda())
for _ in range(3):
    gmg.run_cycle()
torch.cuda.synchronize()
if os.environ.get("NCU"):     # ncu --profile-from-start off: capture this one cycle only
    torch.cuda.profiler.start()
    gmg.run_cycle()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    sys.exit(0)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    gmg.run_cycle()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
tot = sum(e.device_time_total for e in ev)
print(f"one V-cycle: {tot / 1e3:.3f} ms device over {len(ev)} kernels")
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    nm = e.name.replace("pff::(anonymous namespace)::", "").replace("void ", "").split("(")[0]
    agg[nm[:60]][0] += 1
    agg[nm[:60]][1] += e.device_time_total
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {t:9.1f} us  x{c:4d}  {k}")
print("launch sequence (us):")
for e in ev:
    nm = e.name.replace("pff::(anonymous namespace)::", "").replace("void ", "").split("(")[0]
    print(f"  {e.device_time_total:8.1f}  {nm[:70]}")
