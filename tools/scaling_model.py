"""Strong-scaling model of the configs[4] Newton-step solve (GMRES(50) + GMG,
4096^2 Q2) over N B200s with the slab V-cycle of distributed.py.

Inputs are single-GPU MEASUREMENTS (profiles/r02/vcycle_levels_l12.json from
tools/prof_vcycle_levels.py): per level the V-cycle's device time split into
a size-proportional part and a per-level floor (the small levels' serial
kernel chains), plus the operator and orthogonalisation time per GMRES
iteration.  Per slab level the proportional part divides by N, the floor does
not; every slab-level operator application adds a ghost-row exchange (NCCL P2P
over NVLink: latency t_msg + bytes / bw, half of it hidden behind the interior
rows); the restriction adds one reverse message and the prolongation one
exchange; the agglomerated levels run redundantly on every rank after one
all-reduce; GMRES adds three all-reduces per iteration (CGS2 + norm).

    python tools/scaling_model.py profiles/r02/vcycle_levels_l12.json
"""

import json
import sys

T_MSG = 15e-6          # NCCL P2P / all-reduce small-message latency over NVLink (s)
BW = 900e9             # NVLink 5 per direction (B/s)
HIDDEN = 0.5           # share of the halo latency hidden behind interior rows
APPLIES = 14           # operator applications per slab level per V-cycle (sweeps 3)


def slab_levels(finest, n_gpu, min_rows=16, coarse=2):
    """The levels distributed.DistributedGmg puts in slabs."""
    out = [finest]
    while True:
        l = out[-1] - 1
        if l - 1 < coarse or 2 ** l < 64 or 2 ** l // n_gpu < max(min_rows, 2):
            return out
        out.append(l)


def model(d, n_gpu):
    levels = {L["level"]: L for L in d["levels"]}
    finest = max(levels)
    slab = slab_levels(finest, n_gpu) if n_gpu > 1 else sorted(levels, reverse=True)
    t_v = 0.0
    for l, L in levels.items():
        if n_gpu > 1 and l in slab:
            np1 = 2 * 2 ** l + 1
            halo = T_MSG + 3 * 3 * np1 * 8 / BW          # p + 1 rows x 3 components
            comm = APPLIES * halo * (1 - HIDDEN) + 2 * halo
            t_v += L["floor_s"] + L["prop_s"] / n_gpu + comm
        else:
            t_v += L["floor_s"] + L["prop_s"]              # 1 GPU, or agglomerated (redundant)
    if n_gpu > 1:
        t_v += T_MSG                                       # the agglomeration all-reduce
    t_it = t_v + d["operator_s"] / n_gpu + d["ortho_s"] / n_gpu + (3 * T_MSG if n_gpu > 1 else 0.0)
    return {"n_gpus": n_gpu, "slab_levels": slab if n_gpu > 1 else [],
            "vcycle_ms": round(1e3 * t_v, 3), "iteration_ms": round(1e3 * t_it, 3),
            "gmres_s": round(d["iterations"] * t_it, 3)}


def main(path):
    with open(path) as f:
        d = json.load(f)
    base = model(d, 1)
    out = []
    for n in (1, 2, 4, 8):
        r = model(d, n)
        r["speedup"] = round(base["gmres_s"] / r["gmres_s"], 2)
        out.append(r)
        print(json.dumps(r))
    return out


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02/vcycle_levels_l12.json")
