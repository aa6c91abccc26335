import os, sys
from collections import defaultdict
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
import paper_2005_00331_b200 as P
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe", seed=0, notch=True)
def mk():
    st = P.LinearizationState(h, 10, params, split="miehe")
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    return st
gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
for _ in range(2):
    st = mk(); st.refresh_cache(); gmg.setup(st); gmg.run_cycle(); torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
st = mk()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    st.refresh_cache(); gmg.setup(st); gmg.run_cycle()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    nm = e.name.replace("pff::(anonymous namespace)::", "").replace("void ", "").split("(")[0][:60]
    agg[nm][0] += 1; agg[nm][1] += e.device_time_total
tot = sum(v[1] for v in agg.values())
print(f"setup device total {tot/1e3:.2f} ms over {len(ev)} kernels")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {t/1e3:8.3f} ms x{c:5d}  {k}")
