cd $GRAFT_REPO_ROOT
for mode in 0 1 0 1; do
for r in "1,2,4,4,4,4,4,4,2,1" "1,2,3,3,3,3,3,3,3,3,2,1" "1,1,2,2,2,2,2,2,2,2,2,2,2,2,1,1" "2,4,6,6,6,4,2"; do
PFF_PIPE_1D=$mode PFF_PIPE_RAMP=$r taskset -c $(python -c "import bench;c=bench.gpu_local_cpus(0);print(','.join(map(str,sorted(c))) if c else '0-7')") timeout 200 python - <<'P'
import os, time, torch, bench, paper_2005_00331_b200 as P
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe")
st = P.LinearizationState(h, 10, params, split="miehe")
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act); st.set_dirichlet_nodes(dirn)
st.refresh_cache()
xh = torch.from_numpy(x).pin_memory()
for _ in range(3): yh = P.apply_jacobian(st, xh)
torch.cuda.synchronize(); best = []
for rep in range(3):
    t0 = time.perf_counter()
    for _ in range(20): yh = P.apply_jacobian(st, xh)
    torch.cuda.synchronize(); best.append((time.perf_counter() - t0) / 20)
print("1d" if os.environ["PFF_PIPE_1D"]=="1" else "2d", os.environ["PFF_PIPE_RAMP"], " ".join(f"{x.size/t/1e9:.3f}" for t in best), "GDoF/s", flush=True)
P
done; done
