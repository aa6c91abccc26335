"""cProfile of a warm GmgPreconditioner.setup on configs[3] (the bench's pattern:
a fresh state, the preconditioner object re-used), by own and cumulative time."""
import cProfile
import io
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402

h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe", seed=0, notch=True)
gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
for rep in range(3):
    st = P.LinearizationState(h, 10, params, split="miehe")
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act); st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    gmg.setup(st)
    torch.cuda.synchronize()
    pr.disable()
for key in ("tottime", "cumulative"):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats(key).print_stats(25)
    print(s.getvalue()[:6000])
