"""Device timeline of one e2e apply_jacobian call (pinned host in/out,
configs[1]): start/end of every copy and kernel relative to the first one."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402

h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe")
st = P.LinearizationState(h, 10, params, split="miehe")
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
st.set_dirichlet_nodes(dirn)
st.refresh_cache()
xh = torch.from_numpy(x).pin_memory()
for _ in range(5):
    y = P.apply_jacobian(st, xh)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    y = P.apply_jacobian(st, xh)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{(e.time_range.start - t0):8.1f} {(e.time_range.end - t0):8.1f}  {e.name[:60]}")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
cpu.sort(key=lambda e: e.time_range.start)
print("host span", (cpu[-1].time_range.end - cpu[0].time_range.start), "us")
