#!/usr/bin/env python
"""Benchmark of the sparse-grid dG streamline-diffusion strip solver on B200.

A "step" is one time strip of the paper's method (eq. (4)): the jump
and inflow load, the Richardson iteration with the combination-technique
preconditioner (l.540-566) whose block solves apply the per-grid strip
operator sum_t T_t (x) A_t (x) B_t (the hot path), the cross-grid residual,
and the trace.  Metric: strip-operator DOF-applies/s (whole job), plus time
steps/s and the roofline of the strip-operator kernels.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl reference]

N > 1 runs N independent replicas ("replicas only": the method does not
shard), one per rank under torchrun; value = sum over ranks.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = "c4_6d_stream"
METRIC = "strip-operator DOF-applies/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--L", type=int, default=None, help="override combination level (not a bench line)")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--rtol", type=float, default=1e-10)
    ap.add_argument("--inner-rtol", type=float, default=1e-2)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--secondary", default="c2_4d_stream",
                    help="second workload measured in the same run (configs[2], the largest); 'none' to skip")
    ap.add_argument("--secondary-steps", type=int, default=2)
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.check_output(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                               "--format=csv,noheader,nounits"], timeout=5).decode().strip()
                self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(s[0]) for s in self.samples)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if "Active" in v and "Not" not in v:
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]), "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def apply_traffic(workload):
    """Measured DRAM bytes per DOF-apply of the strip-operator apply for this workload,
    from the committed ncu capture (tools/apply_traffic.py -> profiles/apply_traffic.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "apply_traffic.json")))[workload]
    except Exception:
        return None


def combine_ranks(ms, dof, world, device="cpu"):
    """Replicas-only aggregation: time = max over ranks,
    work = sum over ranks.  Host logic, tested with gloo on CPU."""
    if world <= 1:
        return ms, dof
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms, dof], dtype=torch.float64, device=device)
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx[0]), float(sm[1])


def cpu_baseline(cfg_name, budget_s=15.0):
    """The oracle (unmodified) timed on the host cores on a bounded sample of the
    same workload: strip-operator applies on the component grids of the same
    configuration family at a reduced combination level (sample stated)."""
    import numpy as np
    from oracle.sgrid import SGProblem
    from sginputs import get_config
    L0 = {"c0_2d_const": 6, "c1_2d_rot": 10, "c2_4d_stream": 7, "c3_4d_lshape": 6, "c4_6d_stream": 5}[cfg_name]
    cfg = get_config(cfg_name, L=L0)
    o = SGProblem(cfg, galerkin="direct")
    rng = np.random.default_rng(0)
    X = {l: rng.standard_normal(o.shape(l)) for l in o.active}
    for l in o.active:        # assembly outside the timed region
        o.apply_diag(l, X[l])
    dof = 0
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < budget_s or n == 0:
        for l in o.active:
            o.apply_diag(l, X[l])
            dof += int(np.prod(o.shape(l)))
        n += 1
    dt = time.perf_counter() - t0
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count()
    return {"value": dof / dt, "unit": "DOF-applies/s", "cores": cores, "kind": "oracle",
            "sample": f"oracle apply_diag over all {len(o.active)} active grids of {cfg_name} at L={L0} "
                      f"({sum(int(np.prod(o.shape(l))) for l in o.active)} DOF/sweep), {n} sweeps, {dt:.1f}s",
            "threads_note": "numpy/scipy default threading"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cb = cpu_baseline(args.config, budget_s=max(5.0, 20.0 / max(args.steps, 1)))
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "DOF-applies/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "dtype": "f64", "data": "synthetic", "vs_baseline": None,
            "config": {"workload": args.config, "note": "oracle on host cores, bounded sample"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "DOF-applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def fp64_peak():
    """Measured FP64 peaks of this GPU: tools/fp64_peak (DFMA register chains on every SM and
    DMMA mma.sync.m8n8k4), run live; fallback: the committed profiles/fp64_peak.json of an
    earlier run on this pool; last resort: derived from the guide's unit counts."""
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    try:
        out = subprocess.check_output([exe], timeout=60).decode().strip().splitlines()[-1]
        d = json.loads(out)
        d["source"] = "tools/fp64_peak, measured live on this GPU (" + d.get("how", "") + ")"
        return d
    except Exception:
        pass
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        d["source"] = "profiles/fp64_peak.json (tools/fp64_peak on an earlier box of this pool)"
        return d
    except Exception:
        sm_max = (peaks().get("sm_max_mhz") or 1965.0) / 1e3
        return {"dfma_tflops": 148 * 64 * 2 * sm_max / 1e3, "source": "derived: 148 SM x 64 FMA/clk x 2 x sm_max"}


def measure(args, cfg, world, steps, warmup, e2e_steps, timing=True):
    """Warm up, then time `steps` strips of the workload (device events on the handle's stream,
    barrier + synchronize on both sides, max over ranks).  Strips run in order j = 1..N
    (N = round(T/tau)) and start again from the interpolated u0 after the final time T."""
    import torch
    import torch.distributed as dist
    from paper_2204_05988_b200 import Problem
    stream = torch.cuda.current_stream()
    t_setup = time.perf_counter()
    prob = Problem(cfg, stream=stream)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    N = int(round(cfg["T"] / cfg["tau"]))
    n_tr = prob.set_size(0, 1)
    trace = torch.zeros(n_tr, dtype=torch.float64, device="cuda")
    state = {"j": 1}

    def one_strip(tr, host=False):
        if state["j"] > N:                  # past T: the next run of the workload starts at u0
            state["j"] = 1
            if host:
                t = torch.zeros(n_tr, dtype=torch.float64, device="cuda")
                prob.sg_interp_u0(t)
                tr[:] = t.cpu().numpy()
            else:
                prob.sg_interp_u0(tr)
        prob.sg_step(state["j"], 1, tr, args.rtol, args.inner_rtol)
        state["j"] += 1

    prob.sg_interp_u0(trace)
    for _ in range(warmup):
        one_strip(trace)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    prob.reset_stats()
    prob.set_timing(timing)
    j_first = state["j"]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(steps):
            one_strip(trace)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    st = prob.stats()
    kt = prob.kernel_time()
    health = prob.health()
    prob.set_timing(False)
    ms_max, dof_all = combine_ranks(ms, float(st["dof_applied"]), world, device="cuda")
    res = {"ms": ms, "ms_max": ms_max, "dof_all": dof_all, "stats": st, "kt": kt, "health": health,
           "clocks": clk.summary(), "setup_s": t_setup, "N": N, "strips": [j_first, state["j"] - 1],
           "prob": prob, "n_tr": n_tr}
    # ------------------------------------------------------------- e2e (host buffers)
    if e2e_steps > 0:
        import numpy as np
        host = torch.empty(n_tr, dtype=torch.float64).pin_memory()
        host.copy_(trace)
        hnp = host.numpy()
        prob.reset_stats()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            one_strip(hnp, host=True)       # sg_step(host trace): H2D trace, strip, D2H trace
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t[0])
        st2 = prob.stats()
        dof2 = float(st2["dof_applied"]) * world
        res["e2e"] = {"value": dof2 / dt, "unit": "DOF-applies/s", "h2d_bytes_per_step": 8 * n_tr,
                      "d2h_bytes_per_step": 8 * n_tr, "time_steps_per_s": e2e_steps * world / dt,
                      "steps": e2e_steps,
                      "note": "sg_step(host trace): H2D trace, strip solve, D2H trace; host wall clock"}
    return res


def roofline(res, cfg, fp):
    """Roofline of the strip-operator apply (one 'launch' = one apply on one component grid,
    all its kernels), from the device timestamps around every apply inside the timed region."""
    kt, st, ms = res["kt"], res["stats"], res["ms"]
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    peak_tf = fp["dfma_tflops"]
    sec = kt["ms"] / 1e3
    achieved_tf = (kt["flops"] / 1e12) / sec if sec > 0 else None
    achieved_gbs = (kt["bytes"] / 1e9) / sec if sec > 0 else None
    n_ap = max(kt["launches"], 1)
    roof = {"bound": "alu", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
            "frac": (achieved_tf / peak_tf) if achieved_tf else None, "traffic": None,
            "kernel": ("strip-operator apply per component grid (all its kernels): fused k_fwhole on tiny "
                       "x-lattices; else pass 1 along v (k_vmom shifted moments / k_vfan_st stencils) + pass 2 "
                       "along x (k_xfanin_tma TMA line sweep, k_xwhole, k_xgat_st, k_gather_s2c / k_gather_s2); "
                       "device globaltimer stamps around every apply"),
            "peak_source": "FP64 DFMA pipe, " + fp.get("source", ""),
            "flops_note": "2 FLOP per multiply-add on the structural nonzeros of the factor matrices "
                          "(|a_ij| > 1e-12 max|a|), face groups on boundary rows only (DESIGN.md sec. 5)",
            "algorithmic_flops_per_launch": kt["flops"] / n_ap,
            "algorithmic_bytes_per_launch": kt["bytes"] / n_ap,
            "dof_per_launch": float(st["dof_applied"]) / max(st["applies"], 1),
            "hbm_view": {"achieved_gbs": achieved_gbs, "peak_gbs": hbm,
                         "frac": (achieved_gbs / hbm) if achieved_gbs else None,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)" if "hbm_gbs" in pk
                         else "fallback 6650 GB/s",
                         "note": "algorithmic bytes = read X + write Y + the factor data the launched kernels "
                                 "read (class tables / per-column coefficients / ELL arrays)"},
            "dmma_peak_tflops": fp.get("dmma_tflops"),
            "share_of_step": (kt["ms"] / ms) if ms > 0 else None,
            "avg_apply_ms": kt["ms"] / n_ap}
    tr = apply_traffic(cfg["name"])
    if tr and st["applies"]:
        dof_per_apply = float(st["dof_applied"]) / st["applies"]
        roof["traffic"] = tr["dram_bytes_per_dof"] * dof_per_apply
        roof["traffic_note"] = ("ncu dram__bytes_read.sum + dram__bytes_write.sum of the apply kernels, "
                                "%.1f B per DOF-apply (%s) x %.0f DOF per apply of this run"
                                % (tr["dram_bytes_per_dof"], tr["source"], dof_per_apply))
    return roof


def summary(res, cfg, fp, world, steps):
    st = res["stats"]
    value = res["dof_all"] / (res["ms_max"] / 1e3)
    prob = res["prob"]
    return {"value": value, "ms_per_step": res["ms_max"] / steps,
            "time_steps_per_s": steps * world / (res["ms_max"] / 1e3),
            "config": {"workload": cfg["name"], "L": cfg["L"], "d": cfg["d"], "q": cfg["q"], "tau": cfg["tau"],
                       "strips_total": res["N"], "strips_timed": res["strips"],
                       "strips_note": "strips j run in order 1..N (N = round(T/tau)); after T the workload "
                                      "restarts from the interpolated u0",
                       "parallelism": f"replicas{world}",
                       "l2": "inputs larger than L2 (component grids up to %.0f MB)" % (
                           max(prob.grid_info(0, g)[2] * prob.grid_info(0, g)[3] for g in range(prob.num_grids(0)))
                           * 8 * prob.S / 1e6),
                       "dof_active": prob.set_size(0, prob.S)},
            "gpu_launches": st["launches"], "applies": st["applies"], "outer_iters": st["outer_iters"],
            "inner_iters": st["inner_iters"], "outer_mr_switches": st.get("outer_mr_switches"),
            "solver_health": res["health"],
            "setup_s": res["setup_s"], "roofline": roofline(res, cfg, fp), "clocks": res["clocks"]}


def main():
    args = parse()
    if args.secondary == "none":
        args.secondary = None
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch
    import torch.distributed as dist
    from sginputs import get_config

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fp = fp64_peak()
    cfg_over = {} if args.L is None else {"L": args.L}
    cfg = get_config(args.config, **cfg_over)
    res = measure(args, cfg, world, args.steps, args.warmup, 0 if args.no_e2e else args.e2e_steps)
    sm = summary(res, cfg, fp, world, args.steps)
    flagged = any(v for v in res["health"].values())
    out = {"metric": METRIC, "value": sm["value"], "unit": "DOF-applies/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": sm["ms_per_step"], "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": dict(sm["config"], rtol=args.rtol, inner_rtol=args.inner_rtol),
           "time_steps_per_s": sm["time_steps_per_s"],
           "gpu_launches": sm["gpu_launches"], "applies": sm["applies"], "outer_iters": sm["outer_iters"],
           "inner_iters": sm["inner_iters"], "outer_mr_switches": sm["outer_mr_switches"],
           "solver_health": sm["solver_health"], "flagged_unconverged": flagged,
           "setup_s": sm["setup_s"], "roofline": sm["roofline"], "clocks": sm["clocks"], "e2e": res.get("e2e")}
    del res
    # configs[2] (the largest configuration by DOF) measured in the same run, fewer strips
    if args.secondary and args.secondary != args.config and world == 1:
        try:
            cfg2 = get_config(args.secondary)
            r2 = measure(args, cfg2, world, args.secondary_steps, 1, 0)
            s2 = summary(r2, cfg2, fp, world, args.secondary_steps)
            s2["steps"], s2["warmup"] = args.secondary_steps, 1
            s2["solver_health"] = r2["health"]
            out["secondary"] = {args.secondary: s2}
            del r2
        except Exception as ex:
            out["secondary"] = {args.secondary: {"error": str(ex)}}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            out["cpu_baseline"] = cpu_baseline(cfg["name"])
        except Exception as ex:  # never fail the bench line on the baseline leg
            out["cpu_baseline"] = {"error": str(ex)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
