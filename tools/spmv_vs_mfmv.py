"""Assembled SpMV (cuSPARSE, device CSR) versus the matrix-free application
(the paper's MFMV-vs-SpMV comparison) on
the B200: benchmark_vmult over degrees and levels, plus memory_report."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_00331_b200 as P  # noqa: E402

cases = [(1, 8), (1, 10), (2, 7), (2, 9), (2, 10), (4, 6), (4, 8), (4, 9)]
if len(sys.argv) > 1:
    cases = [tuple(int(v) for v in c.split(":")) for c in sys.argv[1:]]
for degree, level in cases:
    cfg = P.ScenarioConfig(scenario="tension", level=level, degree=degree, steps=1,
                           params=P.MaterialParams(eps=2.0 / 2 ** level))
    try:
        recs = P.benchmark_vmult(cfg, reps=20)
    except Exception as e:   # report and continue with the next size
        print(json.dumps({"degree": degree, "level": level, "error": repr(e)[:200]}), flush=True)
        continue
    out = {"degree": degree, "level": level, "dofs": recs[0].dofs}
    for r in recs:
        out[r.kind + "_s"] = r.best_time_s
    if "spmv_s" in out:
        out["mfmv_speedup"] = out["spmv_s"] / out["mfmv_s"]
    mem = P.memory_report(cfg) if level <= 9 else None
    if mem:
        out["csr_B_per_dof"] = round(mem.csr_bytes_per_dof, 1)
        out["mf_B_per_dof"] = round(mem.mf_bytes_per_dof, 1)
    print(json.dumps(out), flush=True)
    torch.cuda.empty_cache()
