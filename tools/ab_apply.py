"""Generic-path (and sweep) applications for a same-box A/B between two builds
(PFF_LIB): a digest of every mode's output (bitwise comparison across runs) and
CUDA-event times (python tools/ab_apply.py [degree level])."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_00331_b200 as P  # noqa: E402
from paper_2005_00331_b200 import _lib  # noqa: E402

p, level = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4, 9)
for split in ("miehe", "none"):
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(p, level, split, seed=0)
    st = P.LinearizationState(h, level, params, split=split)
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    n = st.n_scalar
    xd = torch.from_numpy(x).cuda()
    for mode, name, sl, nout in ((_lib.MODE_FULL, "full", slice(0, 3 * n), 3 * n),
                                 (_lib.MODE_UU, "uu", slice(0, 2 * n), 2 * n),
                                 (_lib.MODE_PHIPHI, "phiphi", slice(2 * n, 3 * n), n),
                                 (_lib.MODE_PHIROW, "phirow", slice(0, 3 * n), n)):
        src = xd[sl].contiguous()
        out = torch.empty(nout, dtype=torch.float64, device="cuda")
        for _ in range(3):
            st.apply_into(mode, src, out)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(50):
            st.apply_into(mode, src, out)
        ev[1].record()
        torch.cuda.synchronize()
        dig = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"Q{p} level {level} {split:6s} {name:7s} {ev[0].elapsed_time(ev[1]) / 50 * 1e3:8.1f} us  {dig}",
              flush=True)
