import sys, os, time, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_2005_00331_b200 as P
from paper_2005_00331_b200 import operator as OP
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe")
st = P.LinearizationState(h, 10, params, split="miehe")
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act); st.set_dirichlet_nodes(dirn)
st.refresh_cache()
xh = torch.from_numpy(x).pin_memory()
for K in (1, 2, 4, 8, 16, 32):
    OP._PIPE_CHUNKS = K
    for _ in range(3): y = P.apply_jacobian(st, xh)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): y = P.apply_jacobian(st, xh)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
    print(f"K={K}: {dt*1e3:.2f} ms/call  {3*st.n_scalar/dt/1e9:.2f} GDoF/s")
# timeline of one call
OP._PIPE_CHUNKS = 8
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    y = P.apply_jacobian(st, xh); torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start)[:60]:
    print(f"{(e.time_range.start-t0)/1e3:8.3f} ms  {(e.time_range.end-e.time_range.start)/1e3:7.3f} ms  {e.name[:40]}")
