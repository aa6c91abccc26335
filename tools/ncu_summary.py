"""Summarise an .ncu-rep (raw metrics + top stall reasons + hottest SASS)."""
import csv
import io
import subprocess
import sys
from collections import Counter

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def main(rep, top=15):
    r = raw(rep)
    print(f"# {rep}")
    for k in WANT:
        if k in r:
            print(f"{k:70s} {r[k][0]} {r[k][1]}")
    st = [(float(v[0]), k) for k, v in r.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(v for v, _ in st) or 1
    print("## stall samples (share)")
    for v, k in sorted(st, reverse=True)[:8]:
        print(f"  {100 * v / tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    isrc, iw = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")

    def num(x):
        try:
            float(x[iw] or 0)
            return True
        except (ValueError, IndexError):
            return False
    # several captured launches repeat the header: keep the numeric rows only
    data = [x for x in rows[2:] if num(x)]
    tot = sum(float(x[iw] or 0) for x in data) or 1
    c = Counter()
    for x in data:
        toks = x[isrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        c[op.split(".")[0]] += float(x[iw] or 0)
    print("## stall samples by opcode")
    print("  " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in c.most_common(12)))
    print("## hottest instructions")
    for x in sorted(data, key=lambda x: -float(x[iw] or 0))[:top]:
        print(f"  {100 * float(x[iw]) / tot:5.2f}%  {x[isrc][:80]}")


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
