import cProfile, pstats, sys, os, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_2005_00331_b200 as P
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe", seed=0, notch=True)
for rep in range(2):
    st = P.LinearizationState(h, 10, params, split="miehe")
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act); st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    pr = cProfile.Profile()
    pr.enable()
    gmg.setup(st)
    torch.cuda.synchronize()
    pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18)
print(s.getvalue()[:5000])
