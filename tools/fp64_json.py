"""Fold the per-kernel ncu metric CSVs of tools/fp64_run.sh (gpurun_out/fp64_ncu_<tag>.csv, or
the paths given) into profiles/ncu_fp64.json and the FULL-application DRAM bytes of the Q2
configs into profiles/ncu_traffic.json:  python tools/fp64_json.py [csv ...]"""
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
paths = sys.argv[1:] or sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "fp64_ncu_*.csv")))
out_p = os.path.join(ROOT, "profiles", "ncu_fp64.json")
out = json.load(open(out_p)) if os.path.exists(out_p) else {}
for p in paths:
    tag = os.path.basename(p)[len("fp64_ncu_"):-len(".csv")]
    lines = open(p).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    ker = {}
    for r in csv.DictReader(lines[start:]):
        name = r["Kernel Name"].split("void ")[-1].split("(")[0]
        ker.setdefault((r["ID"], name), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    d = {}
    for (_, name), m in ker.items():   # the last launch of each kernel wins (they are identical)
        pre = "smsp__sass_thread_inst_executed_op_"
        d[name] = {
            "fp64_thread_inst": int(m[pre + "dfma_pred_on.sum"] + m[pre + "dadd_pred_on.sum"] +
                                    m[pre + "dmul_pred_on.sum"]),
            "dfma": int(m[pre + "dfma_pred_on.sum"]),
            "dram_bytes": int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]),
            "ncu_us": m["gpu__time_duration.sum"] / 1e3,
            "fp64_pipe_pct_ncu": m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
            "warp_inst": int(m["smsp__inst_executed.sum"]),
        }
    out[tag] = d
    print(tag, json.dumps(d))
json.dump(out, open(out_p, "w"), indent=1)
tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
t = json.load(open(tp))
for split in ("miehe", "none"):
    tag = f"degree2level10split{split}"
    if tag in out:
        t[split] = sum(v["dram_bytes"] for v in out[tag].values())
t["_what"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of k_sweep_q2<FULL> "
              "(apply_jacobian, configs[1] 1024^2 Q2), bytes, from the ncu metric pass of "
              "tools/fp64_run.sh folded by tools/fp64_json.py (profiles/ncu_fp64.json holds the "
              "per-kernel rows); algorithmic bytes per launch = 27 B/DoF x 12,598,275 = 340.2e6")
json.dump(t, open(tp, "w"), indent=1)
