"""Pin the configs[4] Newton-step iteration count with the CPU oracle (test
infrastructure; the oracle is bitwise equal to the reference on every golden
vector and reproduces its GMRES counts, tests/test_oracle_golden.py).

The reference itself (serial numba) cannot run a 4096^2 solve in the build
container (the GMRES(50) basis alone is 82 GB); the oracle on all host threads
of the GPU box can.  Writes tests/golden/pin_oracle_l{level}_{split}.json:
iterations, residual history, Lanczos ranges and a sketch of the first
V-cycle (same sketch as the reference fixtures, tests/conftest.py).

    python tools/pin_newton_oracle.py --level 12 --split miehe
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import sketch  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=12)
    ap.add_argument("--split", default="miehe")
    ap.add_argument("--restart", type=int, default=50)
    ap.add_argument("--out", default=None)
    ap.add_argument("--max-iterations", type=int, default=1000,
                    help="stop after this many GMRES iterations (a bounded pin of the history)")
    args = ap.parse_args()
    nt = O.max_threads()
    t0 = time.perf_counter()
    ost, x = O.baseline_state(2, args.level, args.split, seed=0, notch=True)
    ost.refresh_cache(nthreads=nt)
    n = ost.n
    og = O.Gmg(2, args.level, coarse_level=2, cheb=O.ChebCfg(sweeps=3), nthreads=nt)
    og.setup(ost)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    z = og.apply(x)
    t_v = time.perf_counter() - t0
    sk = {k: v.tolist() for k, v in sketch(z, n).items()}
    del z
    rhs = x.copy()
    rhs[ost.constrained_mask()] = 0.0
    t0 = time.perf_counter()
    res = O.gmres(lambda v: O.apply_jacobian(ost, v, nt), rhs, tol=1e-8,
                  restart=args.restart, preconditioner=og.apply,
                  max_iterations=args.max_iterations)
    t_g = time.perf_counter() - t0
    out = {"level": args.level, "split": args.split, "restart": args.restart,
           "max_iterations": args.max_iterations,
           "iterations": res.iterations, "converged": res.converged,
           "history": [float(v) for v in res.history],
           "ranges": {str(l): [r["uu"][0], r["uu"][1], r["phiphi"][0], r["phiphi"][1]]
                      for l, r in sorted(og.ranges.items())},
           "vcycle_sketch": sk, "threads": nt,
           "seconds": {"setup": round(t_setup, 1), "vcycle": round(t_v, 1), "gmres": round(t_g, 1)},
           "how": "oracle/oracle.py Gmg + gmres (C kernels, OpenMP) on the configs[3]/[4] "
                  "notch inputs, seed 0, sweeps 3, rtol 1e-8"}
    path = args.out or os.path.join(ROOT, "tests", "golden",
                                    f"pin_oracle_l{args.level}_{args.split}.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump(out, f)
    print(json.dumps({k: v for k, v in out.items() if k not in ("history", "vcycle_sketch")}))


if __name__ == "__main__":
    main()
