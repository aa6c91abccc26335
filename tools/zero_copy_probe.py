"""Feasibility probe: the FULL sweep reading x from and writing y to pinned
host memory directly (UVA zero-copy), against the device path."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import _lib  # noqa: E402
L = _lib.load()
h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, 10, "miehe")
st = P.LinearizationState(h, 10, params, split="miehe")
st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act); st.set_dirichlet_nodes(dirn)
st.refresh_cache()
xh = torch.from_numpy(x).pin_memory()
yh = torch.empty_like(xh).pin_memory()
xd = xh.cuda(); yd = torch.empty_like(xd)
s = torch.cuda.current_stream().cuda_stream
hb = st.bind()
L.pff_apply(hb, 0, xd.data_ptr(), yd.data_ptr(), None, s)
torch.cuda.synchronize()
rc = L.pff_apply(hb, 0, xh.data_ptr(), yh.data_ptr(), None, s)
torch.cuda.synchronize()
print("rc", rc, "equal", torch.equal(yh, yd.cpu()), flush=True)
for _ in range(3):
    L.pff_apply(hb, 0, xh.data_ptr(), yh.data_ptr(), None, s)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    L.pff_apply(hb, 0, xh.data_ptr(), yh.data_ptr(), None, s)
    torch.cuda.current_stream().synchronize()
dt = (time.perf_counter() - t) / 20
print(f"zero-copy FULL: {dt*1e3:.3f} ms, {x.size/dt/1e9:.3f} GDoF/s", flush=True)
for name, a, b in (("src host, dst device", xh, yd), ("src device, dst host", xd, yh)):
    for _ in range(3):
        L.pff_apply(hb, 0, a.data_ptr(), b.data_ptr(), None, s)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        L.pff_apply(hb, 0, a.data_ptr(), b.data_ptr(), None, s)
        torch.cuda.current_stream().synchronize()
    dt = (time.perf_counter() - t) / 20
    print(f"{name}: {dt*1e3:.3f} ms", flush=True)
