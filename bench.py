"""Benchmark of the B200 PFF hot path (BASELINE.json metric).

Headline (N=1): configs[1] -- the fp64 Jacobian vmult (apply_jacobian) on the
1024x1024 Q2 mesh, 12,598,275 DoFs, BASELINE value distributions; a step is
one application over the whole vector; value = GDoF/s.  Each step moves
340 MB (> 126 MB L2), so no L2 flush is needed between steps.

Also reported (BASELINE.json's second metric): the GMRES+GMG solve time of
one semi-smooth Newton step on configs[3] (1024^2 Q2, notch phase field,
9 levels, Chebyshev sweeps=3, restart 50, rtol 1e-8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--split miehe|none]
    python bench.py --impl reference ...   # the CPU oracle port on host cores

N>1 (torchrun): the same global problem is split into cell-row slabs, one per
rank (paper_2005_00331_b200/parallel.py); a step is the NCCL ghost-row
exchange plus the slab application -- strong scaling.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_DOF = 27.0   # src+dst 6 + nodal state 4 doubles + 1 flag byte per node / 3


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_peak():
    """Measured FP64 issue peak (tools/micro/dfma_peak.cu -> profiles/fp64_peak.json):
    DFMA thread-instructions per second over the whole GPU."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["dfma_per_s"]), "measured (profiles/fp64_peak.json, tools/micro/dfma_peak.cu)"
    except Exception:
        return 148 * 64 * 1.965e9, "fallback (148 SMs x 64 FP64 lanes x 1.965 GHz)"


def fp64_counts(tag):
    """FP64 thread-instructions (DFMA + DADD + DMUL) per launch of each kernel of
    one application, from the committed ncu capture (profiles/ncu_fp64.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_fp64.json")) as f:
            d = json.load(f)[tag]
        return sum(v["fp64_thread_inst"] for v in d.values()), sum(v["dram_bytes"] for v in d.values())
    except Exception:
        return None, None


def fp64_roof(tag, ms):
    """FP64 pipe fraction of one application: its ncu-counted FP64 instructions
    over its measured time, against the measured DFMA issue peak."""
    inst, _ = fp64_counts(tag)
    pk, src = fp64_peak()
    if inst is None:
        return None
    ach = inst / (ms * 1e-3)
    return {"bound": "fp64", "achieved": round(ach / 1e12, 3), "peak": round(pk / 1e12, 3),
            "unit": "T FP64 inst/s", "frac": round(ach / pk, 4),
            "inst_per_launch": inst, "peak_source": src,
            "counted": "smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on (ncu, "
                       "profiles/ncu_fp64.json)"}


def workload_config(args, ws):
    """The `config` object of both arms (ours and --impl reference)."""
    level, dofs = args.level, 3 * ((2 * 2 ** args.level + 1) ** 2 + 2 ** args.level)
    return {"workload": f"configs[1]: {2 ** level}x{2 ** level} Q2 apply_jacobian, {dofs:,} DoFs",
            "split": args.split, "degree": 2, "level": level, "dofs": dofs,
            "l2": f"inputs larger than L2 ({27 * dofs / 1e6:.0f} MB per step), no flush",
            "parallelism": f"cell-row slabs x{ws}, NCCL ghost-row exchange per step"
                           if ws > 1 else "single GPU"}


def baseline_inputs(p, level, split, seed=0, notch=False):
    """BASELINE.json synthetic draws: u0 ~ U[-1e-3,1e-3] (2n),
    phi0 ~ U[0,1] (n) or the notch profile, x ~ U[-1,1] (3n);
    phi_tilde = phi_old = phi0, active = phi0 < 0.05, Dirichlet = top+bottom."""
    import paper_2005_00331_b200 as P
    h = P.build_hierarchy(level, p)
    dm = h.dof_map(level)
    n = dm.n_scalar
    eps = 2.0 / 2 ** level
    params = P.MaterialParams(lame_lambda=121.15e3, mu=80.77e3, g_c=2.7, kappa=1e-10, eps=eps)
    rng = np.random.default_rng(seed)
    u0 = rng.uniform(-1e-3, 1e-3, 2 * n)
    if notch:
        c = dm.coords
        dx = np.maximum(c[:, 0] - 0.5, 0.0)
        phi0 = 1.0 - np.exp(-np.sqrt(dx * dx + (c[:, 1] - 0.5) ** 2) / eps)
    else:
        phi0 = rng.uniform(0.0, 1.0, n)
    x = rng.uniform(-1.0, 1.0, 3 * n)
    dirichlet = np.unique(np.concatenate([dm.boundary_nodes["top"], dm.boundary_nodes["bottom"]]))
    return h, params, np.concatenate([u0, phi0]), phi0, phi0 < 0.05, dirichlet, x


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index=0, period=0.01):
        self.samples, self.reasons, self.period = [], set(), period
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = nvml_handle(pynvml, index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:   # pragma: no cover - no NVML
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def nvml_handle(pynvml, device: int):
    """NVML handle of CUDA device `device`, found by its PCI bus id: NVML's own
    indices ignore CUDA_VISIBLE_DEVICES and CUDA's device order."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(device)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
    except Exception:
        return pynvml.nvmlDeviceGetHandleByIndex(device)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def traffic_from_profiles(split):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(split)
    except Exception:
        return None


# ----------------------------------------------------------------- ours

def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2005_00331_b200 as P
    from paper_2005_00331_b200 import _lib

    ws, rank, local = dist_env()
    # PFF_BENCH_ONE_GPU=1: every rank on cuda:0 with gloo ghost exchange -- a
    # functional check of the N>1 path on a one-GPU box (ranks never wait on
    # each other inside a kernel); timings from it are not scaling numbers
    one_gpu = os.environ.get("PFF_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if ws > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = _lib.load()
    dev = torch.device("cuda", local)

    p, level = 2, args.level
    h, params, U, pt, act, dirn, x = baseline_inputs(p, level, args.split, seed=0)
    n = h.dof_map(level).n_scalar
    dofs = 3 * n                      # global DoFs of the whole job
    stream = torch.cuda.current_stream()
    if ws == 1:
        st = P.LinearizationState(h, level, params, split=args.split)
        st.set_solution(U)
        st.set_phi_tilde(pt)
        st.set_phi_old(pt)
        st.set_active(act)
        st.set_dirichlet_nodes(dirn)
        st.refresh_cache()
        xd = torch.from_numpy(x).to(dev)
        yd = torch.empty_like(xd)

        def step():
            st.apply_into(_lib.MODE_FULL, xd, yd)
    else:
        # strong scaling: the same global problem in cell-row slabs, one per rank;
        # a step = ghost-row exchange (NCCL send/recv) + the slab application
        from paper_2005_00331_b200.parallel import SlabPartition, SlabState
        part = SlabPartition(p, level, ws)
        dmask = np.zeros(n, dtype=bool)
        dmask[dirn] = True
        st = SlabState(part, rank, params, args.split, U, pt, act, dmask, device=dev)
        st.refresh_cache()
        xd = torch.from_numpy(part.scatter(x, rank, 3)).to(dev)
        yd = st.empty(3)

        def step():
            st.apply_into(_lib.MODE_FULL, xd, yd)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    c0 = L.pff_launch_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = L.pff_launch_counter() - c0
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / args.steps
    value = dofs * args.steps / (ms * 1e-3) / 1e9

    # end to end through the public API with pinned host buffers
    e2e_steps = max(3, min(20, args.steps))
    # the e2e host side runs on the GPU's NUMA node (its pinned buffers are
    # first-touched there); the affinity is restored before the CPU baseline
    aff0 = os.sched_getaffinity(0)
    local_cpus = gpu_local_cpus(local)
    try:
        if local_cpus:
            os.sched_setaffinity(0, local_cpus)
        if ws == 1:
            xh = torch.from_numpy(x).pin_memory()
            for _ in range(3):            # warm the pinned-buffer cache with the timed loop's
                yh = P.apply_jacobian(st, xh)   # pattern (previous result alive: two blocks)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                yh = P.apply_jacobian(st, xh)
            torch.cuda.synchronize()
            e2e_s = (time.perf_counter() - t0) / e2e_steps
            h2d = d2h = 8 * dofs
            # correctness of the timed output (bench never reports an unchecked number)
            yref = P.apply_jacobian(st, xd)
            assert torch.equal(yref, yd)
            assert torch.equal(yh.to(dev), yd)
        else:
            xh = xd.cpu().pin_memory()
            yh = torch.empty(yd.shape, dtype=torch.float64, pin_memory=True)
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                xd.copy_(xh, non_blocking=True)
                st.apply_into(_lib.MODE_FULL, xd, yd)
                yh.copy_(yd)
            torch.cuda.synchronize()
            t = torch.tensor([time.perf_counter() - t0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item()) / e2e_steps
            h2d = d2h = 8 * 3 * st.ln
    finally:
        os.sched_setaffinity(0, aff0)
    # the same kernel timed alone (50 launches after the PCIe-bound e2e loop): the
    # 2000-step headline runs into the power cap, MEASURED_PEAKS' copy peak is a
    # burst figure -- both fractions are reported, `frac` stays the sustained one
    burst = None
    if ws == 1:
        torch.cuda.synchronize()
        time.sleep(0.5)
        for _ in range(3):
            step()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(50):
            step()
        b1.record(stream)
        torch.cuda.synchronize()
        bms = b0.elapsed_time(b1) / 50
        burst = {"steps": 50, "ms_per_step": round(bms, 5),
                 "value": round(dofs / (bms * 1e-3) / 1e9, 3)}
    # the other split's vmult on the same inputs (N=1; not the headline: the
    # reference default is Miehe), CUDA events over 200 applications
    other = None
    if ws == 1 and args.other_split:
        osp = "none" if args.split == "miehe" else "miehe"
        so = P.LinearizationState(h, level, params, split=osp)
        so.set_solution(U)
        so.set_phi_tilde(pt)
        so.set_phi_old(pt)
        so.set_active(act)
        so.set_dirichlet_nodes(dirn)
        so.refresh_cache()
        for _ in range(max(3, args.warmup)):
            so.apply_into(_lib.MODE_FULL, xd, yd)
        reps = 200
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            so.apply_into(_lib.MODE_FULL, xd, yd)
        e1.record(stream)
        torch.cuda.synchronize()
        oms = e0.elapsed_time(e1) / reps
        ov = dofs / (oms * 1e-3) / 1e9
        opk, _ = peaks()
        other = {"split": osp, "value": round(ov, 3), "unit": "GDoF/s", "ms_per_step": round(oms, 5),
                 "steps": reps, "roofline_frac": round(BYTES_PER_DOF * ov / opk, 4),
                 "traffic": traffic_from_profiles(osp)}
        del so
    q4 = None
    if ws == 1 and args.q4:
        try:
            q4 = q4_section(args, P, torch, _lib, stream)
        except Exception as e:   # reported, never silently dropped
            q4 = {"error": f"{type(e).__name__}: {e}"}
    newton = None
    if args.newton:
        # the vmult state (tangent caches, vectors) is not needed any more: give its
        # device memory back before the solver hierarchy and Krylov basis are built
        del st, xd, yd
        release_device_memory(torch)
        try:
            newton = (newton_step_ours(args, P, torch) if ws == 1
                      else newton_step_distributed(args, P, torch, ws, rank, dev))
        except Exception as e:   # reported, never silently dropped
            newton = {"error": f"{type(e).__name__}: {e}"}
        if ws == 1 and rank == 0 and not args.no_cpu_baseline and isinstance(newton, dict) \
                and "iterations" in newton:
            newton["cpu_baseline"] = newton_cpu_baseline(args, newton["iterations"])
    newton4 = None
    if ws == 1 and args.configs4 and args.newton_level != 12:
        # configs[4] (4096^2 Q2, 201 M DoFs) on this one GPU: the N=1 point of the
        # scaling case (bench.py --gpus N runs it over N slabs)
        release_device_memory(torch)
        try:
            a4 = argparse.Namespace(**vars(args))
            a4.newton_level = 12
            newton4 = newton_step_ours(a4, P, torch, warm_runs=False)
        except Exception as e:
            newton4 = {"error": f"{type(e).__name__}: {e}"}
        release_device_memory(torch)

    if rank != 0:
        return
    peak, peak_src = peaks()
    achieved = BYTES_PER_DOF * dofs / ws / (ms_step * 1e-3) / 1e9   # per GPU
    # the CPU baseline is an N=1 figure (rank 0 at N=1 only); the N>1 lines skip it
    cpu = cpu_baseline(args) if (not args.no_cpu_baseline and ws == 1) else None
    out = {
        "metric": "GDoF/s of fp64 Jacobian vmult (apply_jacobian, 1024^2 Q2)",
        "value": round(value, 3),
        "unit": "GDoF/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 5),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE.json configs[1] draws, seed 0)",
        "config": workload_config(args, ws),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic_from_profiles(args.split),
                     "algorithmic_bytes_per_dof": BYTES_PER_DOF, "peak_source": peak_src,
                     "fp64": fp64_roof(f"degree2level10split{args.split}", ms_step)
                             if (ws == 1 and level == 10) else None,
                     "burst": dict(burst, frac=round(BYTES_PER_DOF * burst["value"] / peak, 4))
                              if burst else None},
        "e2e": {"value": round(dofs / e2e_s / 1e9, 4), "unit": "GDoF/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "host_cpus": (f"GPU-local NUMA node ({len(local_cpus)} CPUs)" if local_cpus
                              else "process affinity"),
                "path": "paper_2005_00331_b200.apply_jacobian(state, pinned host tensor): "
                "one pff_apply_host call: row-chunked H2D / sweep / D2H pipeline (copy streams driven natively)"
                        if ws == 1 else "SlabState.apply_into with pinned host slab buffers"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if newton is not None:
        out["newton_step"] = newton
    if other is not None:
        out["other_split"] = other
    if q4 is not None:
        out["q4"] = q4
    if newton4 is not None:
        out["newton_step_configs4"] = newton4
    print(json.dumps(out))


def release_device_memory(torch):
    import gc
    gc.collect()                      # solver objects reference each other (cycles)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def q4_section(args, P, torch, _lib, stream):
    """configs[2]: the same operator on 512^2 Q4 cells (12.6 M DoFs, 5-point Gauss),
    100 repeated applications per split (CUDA events), HBM fraction at the same
    27 B/DoF and the FP64 pipe fraction from the ncu-counted FP64 instructions."""
    level, p = 9, 4
    out = {"config": "configs[2]: 512x512 Q4 apply_jacobian, 5-point Gauss", "reps": 100}
    pk, _ = peaks()
    for split in ("miehe", "none"):
        h, params, U, pt, act, dirn, x = baseline_inputs(p, level, split, seed=0)
        st = P.LinearizationState(h, level, params, split=split)
        st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
        st.set_dirichlet_nodes(dirn)
        st.refresh_cache()
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        for _ in range(5):
            st.apply_into(_lib.MODE_FULL, xd, yd)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(100):
            st.apply_into(_lib.MODE_FULL, xd, yd)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 100
        dofs = xd.numel()
        v = dofs / (ms * 1e-3) / 1e9
        _, traffic = fp64_counts(f"degree4level9split{split}")
        out[split] = {"value": round(v, 3), "unit": "GDoF/s", "ms_per_step": round(ms, 5),
                      "dofs": dofs, "hbm_frac": round(BYTES_PER_DOF * v / pk, 4),
                      "traffic": traffic,
                      "fp64": fp64_roof(f"degree4level9split{split}", ms)}
        del st, xd, yd
        release_device_memory(torch)
    return out


def newton_cpu_baseline(args, iterations, budget_iters=2):
    """The Newton-step solve of configs[3] on the host cores with the C oracle
    port (oracle/oracle.py Gmg + gmres, OpenMP cell kernels): the GMG setup
    (Lanczos on every level) timed whole, then `budget_iters` GMRES iterations
    timed; the total is projected to the GPU's iteration count (a bounded
    sample: the whole solve would take minutes)."""
    from oracle import oracle as O
    nt = host_threads()
    t0 = time.perf_counter()
    ost, x = O.baseline_state(2, args.newton_level, args.split, seed=0, notch=True)
    ost.refresh_cache(nthreads=nt)
    og = O.Gmg(2, args.newton_level, coarse_level=2, cheb=O.ChebCfg(sweeps=3), nthreads=nt)
    og.setup(ost)
    t_setup = time.perf_counter() - t0
    rhs = x.copy()
    rhs[ost.constrained_mask()] = 0.0
    t0 = time.perf_counter()
    O.gmres(lambda v: O.apply_jacobian(ost, v, nt), rhs, tol=1e-8, restart=50,
            max_iterations=budget_iters, preconditioner=og.apply)
    t_it = (time.perf_counter() - t0) / budget_iters
    return {"setup_s": round(t_setup, 2), "seconds_per_iteration": round(t_it, 3),
            "projected_total_s": round(t_setup + iterations * t_it, 1),
            "cores": nt, "kind": "port",
            "sample": f"oracle Gmg.setup + {budget_iters} GMRES(50) iterations of configs[3] "
                      f"({args.split}); total projected to {iterations} iterations (the early "
                      "Arnoldi steps are the cheapest: MGS cost grows with j)"}


def newton_step_ours(args, P, torch, warm_runs=True):
    """configs[3]: one Newton step's GMRES+GMG solve on 1024^2 Q2.  A fresh
    linearisation state (from host arrays) every time; the first solve (cold:
    module loads, first graph capture, allocations) is reported as cold_*, then
    three warm solves re-using the preconditioner object -- GmgPreconditioner.setup
    on the new state, as the reference's ActiveSetSolver does every Newton step
    (src/active_set_solver.py:129-145) -- of which the median (setup + GMRES) is
    the steady-state figure a simulation sees every step."""
    level = args.newton_level
    h, params, U, pt, act, dirn, x = baseline_inputs(2, level, args.split, seed=0, notch=True)
    rhs = x.copy()
    dmask = np.zeros(h.dof_map(level).n_scalar, dtype=bool)
    dmask[dirn] = True
    rhs[np.concatenate([dmask, dmask, act])] = 0.0
    rhs_h = torch.from_numpy(rhs).pin_memory()
    sol_h = torch.empty(rhs_h.numel(), dtype=torch.float64, pin_memory=True)

    phases = {}
    keep = {}

    def one():
        st = P.LinearizationState(h, level, params, split=args.split)
        st.set_solution(U)
        st.set_phi_tilde(pt)
        st.set_phi_old(pt)
        st.set_active(act)
        st.set_dirichlet_nodes(dirn)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st.refresh_cache()
        torch.cuda.synchronize()
        ta = time.perf_counter()
        gmg = keep.get("gmg")
        if gmg is None:
            gmg = keep["gmg"] = P.GmgPreconditioner(h, coarse_level=2,
                                                    cheb=P.ChebyshevConfig(sweeps=3))
        gmg.setup(st)
        torch.cuda.synchronize()
        tb = time.perf_counter()
        gmg.io_buffers()[0].zero_()
        gmg.run_cycle()                       # CUDA-graph capture counted as setup
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t0
        phases["refresh_s"] = round(ta - t0, 4)
        phases["gmg_setup_s"] = round(tb - ta, 4)
        phases["graph_capture_s"] = round(t0 + t_setup - tb, 4)
        t1 = time.perf_counter()
        rhs_d = rhs_h.to("cuda", non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = P.gmres_solve(P.JacobianOperator(st), rhs_d,
                            P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                            preconditioner=gmg.apply)
        e1.record()
        sol_h.copy_(res.solution)             # D2H into pinned memory
        torch.cuda.synchronize()
        return res, t_setup, time.perf_counter() - t1, e0.elapsed_time(e1) / 1e3

    n = h.dof_map(level).n_scalar
    # one solve needs ~(70 + 3 (restart + 1)) n doubles; run the cold and the warm
    # solve back to back only when two hierarchies never coexist in doubt
    res, c_setup, c_gmres, t_dev = one()
    t_setup, t_gmres = c_setup, c_gmres
    release_device_memory(torch)
    warm = warm_runs and \
        8 * n * (70 + 3 * 51) < 0.45 * torch.cuda.get_device_properties(0).total_memory
    runs = []
    reuse_s = None
    if warm:
        # steady state: median of three warm solves (host-side timing noise on
        # shared boxes is large; each run's numbers are kept below)
        for _ in range(3):
            runs.append(one() + (dict(phases),))
        # the setup ActiveSetSolver runs when the active set did not change
        # (src/active_set_solver.py:131): ranges re-used, no Lanczos
        st = P.LinearizationState(h, level, params, split=args.split)
        st.set_solution(U)
        st.set_phi_tilde(pt)
        st.set_phi_old(pt)
        st.set_active(act)
        st.set_dirichlet_nodes(dirn)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st.refresh_cache()
        keep["gmg"].setup(st, reuse_eigen=True)
        keep["gmg"].run_cycle()
        torch.cuda.synchronize()
        reuse_s = time.perf_counter() - t0
        del st
        release_device_memory(torch)
        runs.sort(key=lambda r: r[1] + r[2])
        res, t_setup, t_gmres, t_dev, mid_phases = runs[len(runs) // 2]
        phases.clear()
        phases.update(mid_phases)
    roof = newton_floor(n, res.iterations, 1, t_dev)
    cfg = "configs[3]" if level == 10 else ("configs[4]" if level == 12 else f"level {level}")
    return {"config": f"{cfg}: {2 ** level}^2 Q2 notch, levels 2..{level}, sweeps=3, "
                      "restart 50, rtol 1e-8",
            "split": args.split, "iterations": res.iterations, "converged": res.converged,
            "setup_s": round(t_setup, 4), "gmres_s": round(t_gmres, 4),
            "total_s": round(t_setup + t_gmres, 4), "setup_phases": dict(phases),
            "setup_reuse_eigen_s": round(reuse_s, 4) if reuse_s is not None else None,
            "warm_runs_total_s": [round(r[1] + r[2], 4) for r in runs],
            "cold_setup_s": round(c_setup, 4), "cold_gmres_s": round(c_gmres, 4),
            "gmres_device_s": round(t_dev, 4),
            "roofline": roof,
            "final_rel_residual": res.residual_history[-1] / res.residual_history[0],
            "note": ("median of three warm solves (fresh state each, the preconditioner "
                     "object re-setup as ActiveSetSolver does) after a cold one" if warm
                     else "single (cold) solve: two hierarchies would not fit next to each other")
                    + "; gmres_s includes the rhs H2D and solution D2H"}


def newton_step_distributed(args, P, torch, ws, rank, dev):
    """configs[3] / configs[4] over N slabs: the slab finest level, the
    agglomerated coarse V-cycle and CGS2 GMRES of distributed.py; timed as the
    max over ranks (barrier + synchronize on both sides)."""
    import torch.distributed as dist
    from paper_2005_00331_b200.distributed import DistributedGmg, distributed_gmres
    level = args.newton_level
    h, params, U, pt, act, dirn, x = baseline_inputs(2, level, args.split, seed=0, notch=True)
    n = h.dof_map(level).n_scalar
    dmask = np.zeros(n, dtype=bool)
    dmask[dirn] = True
    rhs = x.copy()
    rhs[np.concatenate([dmask, dmask, act])] = 0.0
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gmg = DistributedGmg(h, level, rank, ws, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3),
                         device=dev)
    gmg.setup(params, args.split, U, pt, pt, act, dmask)
    rl_h = torch.from_numpy(gmg.part.scatter(rhs, rank, 3)).pin_memory()
    sol_h = torch.empty(rl_h.numel(), dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    dist.barrier()
    t_setup = time.perf_counter() - t0
    t1 = time.perf_counter()
    rl = rl_h.to(dev, non_blocking=True)
    res = distributed_gmres(gmg, rl, P.KrylovConfig(relative_tolerance=1e-8, restart=50))
    sol_h.copy_(res.solution)                 # D2H into pinned memory
    torch.cuda.synchronize()
    t_gmres = time.perf_counter() - t1
    t = torch.tensor([t_setup, t_gmres], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_setup, t_gmres = (float(v) for v in t.tolist())
    return {"config": f"{'configs[4]: ' if level == 12 else ''}{2 ** level}^2 Q2 notch over {ws} "
                      f"slabs, levels 2..{level} (levels {gmg.slab_levels[-1]}..{level} in slabs, "
                      f"{gmg.agg_level}..2 agglomerated), sweeps=3, restart 50, rtol 1e-8",
            "split": args.split, "iterations": res.iterations, "converged": res.converged,
            "setup_s": round(t_setup, 4), "gmres_s": round(t_gmres, 4),
            "total_s": round(t_setup + t_gmres, 4), "orthogonalisation": "CGS2",
            "roofline": newton_floor(n, res.iterations, ws, t_gmres),
            "final_rel_residual": res.residual_history[-1] / res.residual_history[0],
            "timing": "max over ranks, wall clock around synchronised regions"}


def newton_floor(n, iterations, ngpu, t):
    """HBM floor of the GMRES+GMG solve (SURVEY.md 8(d) fused-minimum dataflow): per fine
    scalar node and GMRES iteration j, 2.53 kB for the V-cycle over all levels (sweeps=3),
    81 B for the operator and 72 (j+2) B for orthogonalisation + normalisation, spread over
    ngpu GPUs' HBM; frac = floor / t (t: the measured solve time)."""
    floor_b = n * sum(2530 + 81 + 72 * (j % 50 + 2) for j in range(iterations))
    peak, _ = peaks()
    floor_s = floor_b / (ngpu * peak * 1e9)
    return {"bound": "hbm", "floor_s": round(floor_s, 4), "frac": round(floor_s / t, 3),
            "peak_gbs": peak, "n_gpus": ngpu,
            "model": "SURVEY.md 8(d) fused-minimum dataflow: per fine node and iteration 2.53 kB "
                     "V-cycle + 81 B operator + 72(j+2) B MGS, over n_gpus x peak"}


# ------------------------------------------------------------ CPU sides

def cpu_baseline(args, budget_s=15.0):
    """The C oracle port on this host's cores, bounded sample of configs[1]."""
    from oracle import oracle as O
    nt = host_threads()
    st, x = O.baseline_state(2, 10, args.split, seed=0)
    st.refresh_cache(nthreads=nt)
    O.apply_jacobian(st, x, nthreads=nt)   # warm
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end and len(times) < 20:
        t0 = time.perf_counter()
        O.apply_jacobian(st, x, nthreads=nt)
        times.append(time.perf_counter() - t0)
    dofs = 3 * st.n
    return {"value": round(dofs / min(times) / 1e9, 5), "unit": "GDoF/s", "cores": nt,
            "kind": "port",
            "sample": f"oracle/pff_oracle.c apply_jacobian on the full 1024^2 Q2 vector "
                      f"({args.split}), best of {len(times)} in a {budget_s:.0f} s budget"}


def gpu_local_cpus(device: int):
    """The host CPUs of the GPU's NUMA node (sysfs local_cpulist of its PCI
    function), or None when it cannot be read."""
    try:
        import pynvml
        pynvml.nvmlInit()
        try:
            bus = pynvml.nvmlDeviceGetPciInfo(nvml_handle(pynvml, device)).busId
        finally:
            pynvml.nvmlShutdown()
        bus = bus.decode() if isinstance(bus, bytes) else bus
        bus = bus.lower()[-12:]                          # dddd:bb:dd.f
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:   # no NVML / sysfs entry: leave the affinity alone
        return None


def host_threads() -> int:
    """Every host core this process may run on (torchrun sets OMP_NUM_THREADS=1,
    which omp_get_max_threads would report)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:   # pragma: no cover - non-Linux
        return max(1, os.cpu_count() or 1)


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    nt = host_threads()
    st, x = O.baseline_state(2, 10, args.split, seed=0)
    st.refresh_cache(nthreads=nt)
    dofs = 3 * st.n
    for _ in range(min(args.warmup, 1)):
        O.apply_jacobian(st, x, nthreads=nt)
    budget = 120.0
    t0 = time.perf_counter()
    done = 0
    while done < args.steps and (time.perf_counter() - t0) < budget:
        O.apply_jacobian(st, x, nthreads=nt)
        done += 1
    el = time.perf_counter() - t0
    value = dofs * done / el / 1e9
    print(json.dumps({
        "impl": "reference",
        "metric": "GDoF/s of fp64 Jacobian vmult (apply_jacobian, 1024^2 Q2)",
        "value": round(value, 5), "unit": "GDoF/s", "n_gpus": ws, "steps": done,
        "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * el / done, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json configs[1] draws)",
        "config": workload_config(args, 1),
        "cpu_baseline": {"value": round(value, 5), "unit": "GDoF/s", "cores": nt, "kind": "port",
                         "sample": f"{done} full applications (capped at {budget:.0f} s)"},
        "e2e": {"value": round(value, 5), "unit": "GDoF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "reference = fracturekit (Python/numba) cannot travel to the GPU box; this arm "
                "times its C restatement oracle/pff_oracle.c (bitwise equal to the reference "
                "on the golden vectors) with all host threads",
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--split", choices=["miehe", "none"], default="miehe")
    ap.add_argument("--no-newton", dest="newton", action="store_false")
    ap.add_argument("--newton-level", type=int, default=None,
                    help="Newton-step mesh level (default: 10 = configs[3] at N=1, "
                         "12 = configs[4] at N>1)")
    ap.add_argument("--no-configs4", dest="configs4", action="store_false",
                    help="N=1: skip the single configs[4] solve beside configs[3]")
    ap.add_argument("--no-q4", dest="q4", action="store_false",
                    help="N=1: skip the configs[2] (512^2 Q4) vmult object")
    ap.add_argument("--level", type=int, default=10, help="vmult mesh level (10 = configs[1])")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-split", dest="other_split", action="store_false",
                    help="skip the other split's vmult (reported beside the headline)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)   # timing rule: at least 3 warm-up steps
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch our own ranks (the driver may also start us
        # under torchrun, in which case WORLD_SIZE is set and must match --gpus)
        import subprocess
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={os.environ.get('MASTER_PORT', '29531')}",
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if ws != args.gpus and not (ws == 1 and args.gpus == 1):
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.newton_level is None:
        args.newton_level = 12 if ws > 1 else 10
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
