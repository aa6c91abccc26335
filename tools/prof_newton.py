"""Per-kernel device-time breakdown of one Newton-step GMRES+GMG solve
(configs[3]) with torch.profiler (CUPTI activity records, no replay)."""
import argparse
import os
import sys
import time
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=10)
ap.add_argument("--split", default="miehe")
a = ap.parse_args()
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, a.level, a.split, seed=0, notch=True)
st = P.LinearizationState(h, a.level, params, split=a.split)
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
st.set_dirichlet_nodes(dirn)
rhs = x.copy()
mask = np.concatenate([st.dirichlet_nodes, st.dirichlet_nodes, st.active])
rhs[mask] = 0.0
rhs_d = torch.from_numpy(rhs).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
st.refresh_cache()
gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
gmg.setup(st)
gmg.io_buffers()[0].zero_(); gmg.run_cycle()
torch.cuda.synchronize()
print(f"setup {time.perf_counter() - t0:.3f} s")
A = P.JacobianOperator(st)
cfg = P.KrylovConfig(relative_tolerance=1e-8, restart=50)
res = P.gmres_solve(A, rhs_d, cfg, preconditioner=gmg.apply)   # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
res = P.gmres_solve(A, rhs_d, cfg, preconditioner=gmg.apply)
torch.cuda.synchronize()
print(f"gmres {time.perf_counter() - t0:.3f} s, {res.iterations} its")
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    res = P.gmres_solve(A, rhs_d, cfg, preconditioner=gmg.apply)
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name
        for key in ("k_sweep_q2", "k_apply_coop", "k_apply_gather", "k_prolong", "k_restrict",
                    "k_cheb_init", "k_cheb_step", "k_cons", "k_axpby", "k_mgs_step",
                    "k_dot_partials", "k_reduce_final", "k_combine", "k_div", "k_zero_cons3",
                    "Memset", "Memcpy", "k_mul"):
            if key in name:
                name = key + ("<" + name.split("<", 1)[1][:12] if "<" in name and key.startswith("k_sweep") else "")
                break
        agg[name][0] += 1
        agg[name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(f"device total {tot / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} kernels")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {t / 1e3:8.2f} ms {100 * t / tot:5.1f}%  x{c:6d}  {k}")
