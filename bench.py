#!/usr/bin/env python
"""bench.py -- the MOREA hot path on B200 (contract in DESIGN.md §6).

Workload (BASELINE.json configs[3], the paper-scale case that fits one GPU):
C4 = 256x256x96 CT-shaped phantom at 1.5 mm, 600-point Delaunay dual-dynamic
mesh (3607 tets), 7 contour pairs, P = 512 solutions per GPU (weak scaling:
N GPUs evaluate N*512 solutions, the C5 configuration at N = 8).

One step = one MO-RV-GOMEA generation batch over every §8(a) row:
  full evaluation of the P solutions (writes the per-tet cache),
  partial evaluation of one FOS colour class (each edge = one group, delta on
  its dependent tets, old contributions from the cache) for all P solutions,
  fold check of the P solutions, and (N > 1) the NCCL all-gather of the
  per-solution outputs.
Units per step = P full + P * G partial solution evaluations.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solution evals/sec (full & partial) at 1/2/4/8 B200; % HBM roofline"
UNIT = "solution evals/s"
P_PER_GPU = 512
CONFIG_INDEX = 4  # synth config C4 == BASELINE.json configs[3]


def workload_config(P_total, G, world, class_index, T):
    return {
        "workload": f"C4 paper-scale: 256x256x96 CT-shaped phantom (1.5 mm), 600-point Delaunay dual mesh "
                    f"({T} tets), 7 contour pairs, P={P_PER_GPU}/GPU (P_total={P_total}); step = full eval + "
                    f"partial eval of FOS colour class {class_index} ({G} edge groups, tet cache) + fold check"
                    + (" + NCCL all-gather" if world > 1 else ""),
        "population_per_gpu": P_PER_GPU,
        "population_total": P_total,
        "partial_groups": G,
        "l2": "flushed between timed steps (256 MiB device write, untimed)",
        "inputs": "seeded synthetic (synth/, SURVEY.md §8(d)); resident in HBM before timing",
    }


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        # one nvidia-smi in loop mode (a sample every 50 ms) rather than one process
        # per sample, so a sub-second timed region still gets several samples
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                           "--format=csv,noheader,nounits", "-lms", "50"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            for line in self._proc.stdout:
                if self._stop.is_set():
                    break
                line = line.strip()
                if line:
                    self.samples.append([v.strip() for v in line.split(",")])
        except Exception:
            pass

    def __enter__(self):
        self._proc = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)  # first sample before the timed region starts
        return self

    def __exit__(self, *a):
        self._stop.set()
        if getattr(self, "_proc", None) is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_summary():
    """k_raster figures from the committed ncu --set full captures (profiles/ncu_summary.json):
    DRAM bytes per launch (the roofline's `traffic`), L2 / L1-tex hit rates and issue
    utilisation per captured launch (full, partial).  Empty dict if absent."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# --------------------------------------------------------------------------- oracle (CPU) legs
def host_cpu():
    """CPU model and hardware threads of the host the oracle runs on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"host_cpu": model, "host_threads": os.cpu_count()}


def oracle_sample(w, plan_req, sols, n_partial):
    """Time the oracle as it stands on a bounded sample: per solution of `sols`,
    1 full + n_partial partial evaluations."""
    from oracle.oracle import Oracle
    go, ch, nv = plan_req
    orc = Oracle.from_workload(w)
    orc.eval(w.offsets[0])  # untimed: builds the oracle's lazy distance-map memo (load-time work)
    t0 = time.perf_counter()
    for sol in sols:
        _, base = orc.eval(w.offsets[sol])
        for g in range(n_partial):
            orc.eval_partial(w.offsets[sol], base, ch[go[g]:go[g + 1]], nv[sol, go[g]:go[g + 1]])
    dt = time.perf_counter() - t0
    return len(sols) * (1 + n_partial) / dt, dt


def run_reference(args, rank, world):
    """--impl reference: the oracle (plain single-thread C, fp64/int128) on this workload."""
    if rank != 0:
        return 0
    from synth import fos_plan, make_workload, partial_request
    w = make_workload(CONFIG_INDEX, P=P_PER_GPU)
    plan = fos_plan(w.tets, w.N)
    req = partial_request(w, plan, "class", args.class_index)
    from oracle.oracle import Oracle
    go, ch, nv = req
    orc = Oracle.from_workload(w)
    orc.eval(w.offsets[0])
    n_part = 4
    times = []
    for it in range(args.warmup + args.steps):
        sol = 1 + it % (w.P - 1)
        t0 = time.perf_counter()
        _, base = orc.eval(w.offsets[sol])
        for g in range(n_part):
            orc.eval_partial(w.offsets[sol], base, ch[go[g]:go[g + 1]], nv[sol, go[g]:go[g + 1]])
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    total = sum(times)
    units = (1 + n_part) * len(times)
    value = units / total
    G = len(go) - 1
    sample = (f"per step: 1 full + {n_part} partial (1-edge groups of FOS class {args.class_index}) "
              f"evaluations of one C4 solution, oracle single-threaded")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(P_PER_GPU * world, G, world, args.class_index, w.T),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         **host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _fin(x):
    """None for a skipped (NaN) breakdown figure."""
    return x if x == x else None


# --------------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--class-index", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the Sobol / repair / mixing breakdown timings (for ncu launch lists)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # contract: at least 3 untimed warm-up steps

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    import torch
    import torch.distributed as dist

    if args.impl == "reference":
        return run_reference(args, rank, world)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2303_04873_b200 import morea
    from paper_2303_04873_b200.distributed import all_gather_records, pack, shard_bounds
    from synth import fos_plan, make_workload, partial_request

    P_total = P_PER_GPU * world
    w = make_workload(CONFIG_INDEX, P=P_total)
    plan = fos_plan(w.tets, w.N)
    go, ch, nv = partial_request(w, plan, "class", args.class_index)
    G = len(go) - 1
    s0, s1 = shard_bounds(P_total, world, rank)
    P = s1 - s0

    ctx = morea.Context.from_workload(w, device=local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream_handle, device=dev)
    T = w.T
    off_d = torch.from_numpy(w.offsets[s0:s1].copy()).to(dev)
    nv_d = torch.from_numpy(nv[s0:s1].copy()).to(dev)
    obj_d = torch.empty((P, 3), dtype=torch.float64, device=dev)
    acc_d = torch.empty((P, 6), dtype=torch.int64, device=dev)
    cache_d = torch.empty((P, T, 4), dtype=torch.float64, device=dev)
    pobj_d = torch.empty((P * G, 3), dtype=torch.float64, device=dev)
    pacc_d = torch.empty((P * G, 6), dtype=torch.int64, device=dev)
    cnt_d = torch.empty(P, dtype=torch.int32, device=dev)
    sev_d = torch.empty(P, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def step():
        ctx.eval_full(off_d, obj_d, acc_d, cache_d)
        ctx.eval_partial(off_d, acc_d, go, ch, nv_d, cache_d, pobj_d, pacc_d)
        ctx.check_folds(off_d, cnt_d, sev_d, None)
        if world > 1:
            with torch.cuda.stream(stream):
                all_gather_records(pack(obj_d, acc_d), P_total)
                all_gather_records(pack(pobj_d, pacc_d), P_total, rows_per_solution=G)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device time, CUDA events on the context stream, L2 flushed between steps)
    ctx.prof_enable(True)
    ctx.prof_read()
    k0 = ctx.kernel_launches()
    times = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        barrier()
    launches = ctx.kernel_launches() - k0
    prof = ctx.prof_read()
    ctx.prof_enable(False)
    t_local = sum(times)
    t_max = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_max = float(t_max.item())
    units = (P_total + P_total * G) * args.steps
    value = units / (t_max / 1e3)

    # separate full / partial throughputs (same inputs, device time, not in the contract value)
    def timed(fn, reps=3):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    t_full = timed(lambda: ctx.eval_full(off_d, obj_d, acc_d, cache_d))
    t_part = timed(lambda: ctx.eval_partial(off_d, acc_d, go, ch, nv_d, cache_d, pobj_d, pacc_d))
    t_part_nc = timed(lambda: ctx.eval_partial(off_d, acc_d, go, ch, nv_d, None, pobj_d, pacc_d))
    # partial-evaluation sweep over FOS sizes (BASELINE.json configs[3]):
    # 1 edge, 4 and 16 edges of colour class `class_index`, the whole class as one
    # group, all points as one group; cached old contributions; k_raster algorithmic
    # GB/s of the call from the kernel's own counters and CUDA events
    sweep = {}
    peak, peak_src = measured_hbm_peak()
    for kind in ("class", "edges4", "edges16", "wholeclass", "all"):
        sgo, sch, snv = partial_request(w, plan, kind, args.class_index)
        sG = len(sgo) - 1
        snv_d = torch.from_numpy(snv[s0:s1].copy()).to(dev)
        spo = torch.empty((P * sG, 3), dtype=torch.float64, device=dev)
        spa = torch.empty((P * sG, 6), dtype=torch.int64, device=dev)
        run = (lambda sgo=sgo, sch=sch, snv_d=snv_d, spo=spo, spa=spa:
               ctx.eval_partial(off_d, acc_d, sgo, sch, snv_d, cache_d, spo, spa))
        run()
        torch.cuda.synchronize()
        ctx.prof_enable(True)
        ctx.prof_read()
        t_k = timed(run)
        sp = ctx.prof_read()
        ctx.prof_enable(False)
        sb = 8 * sp["samples"] + 12 * sp["band_entries"] + 32 * sp["items"]
        gbs = sb / (sp["ms"] / 1e3) / 1e9 if sp["ms"] > 0 else None
        sweep[kind] = {"groups": sG, "points_per_group": round(len(sch) / sG, 2),
                       "evals_per_s": P * sG * 1e3 / t_k, "ms": t_k,
                       "k_raster_gbs": gbs, "k_raster_frac": (gbs / peak) if gbs else None,
                       "samples_per_eval": sp["samples"] / max(sp["launches"], 1) / (P * sG)}
    t_sobol = t_repair = t_mix = float("nan")
    mix_accept_frac = float("nan")
    if not args.no_extras:
        # NEXT-1: the paper's Sobol-in-tetrahedron sample set (App. A.2), rate 1 sample / voxel
        ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
        t_sobol = timed(lambda: ctx.eval_full(off_d, obj_d, acc_d, None))
        ctx.set_sampler(morea.SAMPLER_VOXEL)
        # NEXT-2: fold repair of the whole population (on a copy of the offsets)
        rep_off = off_d.clone()
        fixed_d = torch.from_numpy(w.fixed_axes.astype("uint8")).to(dev)
        t_repair = timed(lambda: ctx.repair(rep_off.copy_(off_d), 2024, fixed_d, s0), reps=1)
        # NEXT-3: optimal mixing of colour class 0 on the device (model: this shard's
        # population mean and covariance per FOS element, one cluster), on copies of the state
        import numpy as _np
        offs_h = w.offsets[s0:s1]
        mus, Ls = [], []
        for g in range(G):
            X = offs_h[:, ch[go[g]:go[g + 1]], :].reshape(offs_h.shape[0], -1).astype(_np.float64)
            C = _np.cov(X.T, bias=True) + 1e-4 * _np.eye(X.shape[1])
            mus.append(X.mean(0))
            Ls.append(_np.linalg.cholesky(C).ravel())
        mu_d = torch.from_numpy(_np.concatenate(mus)).to(dev)
        L_d = torch.from_numpy(_np.concatenate(Ls)).to(dev)
        cl_d = torch.zeros(P, dtype=torch.int32, device=dev)
        ctx.eval_full(off_d, obj_d, acc_d, cache_d)  # voxel-mode state of off_d (the Sobol run overwrote it)
        mx_off, mx_acc, mx_obj, mx_tc = off_d.clone(), acc_d.clone(), obj_d.clone(), cache_d.clone()
        mx_flags = torch.zeros((P, G), dtype=torch.uint8, device=dev)

        def mix_once():
            mx_off.copy_(off_d); mx_acc.copy_(acc_d); mx_obj.copy_(obj_d); mx_tc.copy_(cache_d)
            ctx.mix_class(mx_off, mx_acc, mx_obj, mx_tc, go, ch, cl_d, mu_d, L_d, fixed_d, None, 0.0, 2024, 0, s0,
                          mx_flags)
        mix_once()  # first call allocates the mixing scratch
        t_mix = timed(mix_once, reps=2)
        mix_accept_frac = float(mx_flags.float().mean().item())

    # plain-load path (volumes beyond the 2D gather-texture limits, e.g. 512 x 512 x 128):
    # the same full evaluation with MOREA_NO_TEX on a second context
    t_plain = float("nan")
    if not args.no_extras:
        os.environ["MOREA_NO_TEX"] = "1"
        ctx_plain = morea.Context.from_workload(w, device=local_rank)
        del os.environ["MOREA_NO_TEX"]
        stream_plain = torch.cuda.ExternalStream(ctx_plain.stream_handle, device=dev)
        ctx_plain.eval_full(off_d, obj_d, acc_d, None)
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream_plain)
        for _ in range(3):
            ctx_plain.eval_full(off_d, obj_d, acc_d, None)
        a1.record(stream_plain)
        torch.cuda.synchronize()
        t_plain = a0.elapsed_time(a1) / 3
        ctx_plain.close()

    # ---- roofline of the dominant kernel (k_raster), SURVEY.md §8(d) algorithmic bytes
    alg_bytes = 8 * prof["samples"] + 12 * prof["band_entries"] + 32 * prof["items"]
    achieved = alg_bytes / (prof["ms"] / 1e3) / 1e9 if prof["ms"] > 0 else None
    per_launch_bytes = alg_bytes / max(prof["launches"], 1)
    ncu = ncu_summary()
    traffic = ncu.get("k_raster_dram_bytes_per_launch")

    # ---- e2e: the same step through the C-ABI with HOST buffers (pinned), copies inside
    off_h = torch.from_numpy(w.offsets[s0:s1].copy()).pin_memory()
    nv_h = torch.from_numpy(nv[s0:s1].copy()).pin_memory()
    obj_h = torch.empty((P, 3), dtype=torch.float64).pin_memory()
    acc_h = torch.empty((P, 6), dtype=torch.int64).pin_memory()
    pobj_h = torch.empty((P * G, 3), dtype=torch.float64).pin_memory()
    pacc_h = torch.empty((P * G, 6), dtype=torch.int64).pin_memory()
    cnt_h = torch.empty(P, dtype=torch.int32).pin_memory()
    sev_h = torch.empty(P, dtype=torch.float64).pin_memory()

    def step_e2e():
        ctx.eval_full(off_h, obj_h, acc_h, cache_d)
        ctx.eval_partial(off_h, acc_h, go, ch, nv_h, cache_d, pobj_h, pacc_h)
        ctx.check_folds(off_h, cnt_h, sev_h, None)
        if world > 1:
            with torch.cuda.stream(stream):
                all_gather_records(pack(obj_d, acc_d), P_total)
                all_gather_records(pack(pobj_d, pacc_d), P_total, rows_per_solution=G)
            torch.cuda.synchronize()

    for _ in range(2):
        step_e2e()
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        step_e2e()
        e2e_times.append(time.perf_counter() - t0)
    t_e2e = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = units / float(t_e2e.item())
    h2d = (2 * off_h.numel() * 4 + nv_h.numel() * 4 + acc_h.numel() * 8)
    d2h = (obj_h.numel() + acc_h.numel() + pobj_h.numel() + pacc_h.numel()) * 8 + cnt_h.numel() * 4 + sev_h.numel() * 8

    # ---- CPU baseline: the oracle as it stands on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_part, sols = 8, (1, 2, 3, 4)
        v, dt = oracle_sample(w, (go, ch, nv), sols, n_part)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"solutions 1-4 of this C4 workload, each 1 full + {n_part} partial "
                         f"(1-edge groups, FOS class {args.class_index}) evaluations, single thread, "
                         f"{dt:.1f} s", **host_cpu()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(P_total, G, world, args.class_index, T),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": traffic, "kernel": "k_raster",
                         "algorithmic_bytes_per_launch": per_launch_bytes, "peak_source": peak_src,
                         "launches": prof["launches"], "kernel_ms": prof["ms"],
                         "ncu": {"source": ncu.get("source"), "l2_hit_pct": ncu.get("k_raster_l2_hit_pct"),
                                 "l1tex_hit_pct": ncu.get("k_raster_l1tex_hit_pct"),
                                 "issue_active_pct": ncu.get("k_raster_issue_active_pct"),
                                 "note": "per captured launch (full, cached partial); the kernel is "
                                         "gather-latency bound, DESIGN.md §4.4"}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "breakdown": {
                "full_evals_per_s": P * 1e3 / t_full, "full_ms": t_full,
                "partial_evals_per_s": P * G * 1e3 / t_part, "partial_ms": t_part,
                "partial_nocache_evals_per_s": P * G * 1e3 / t_part_nc,
                "sobol_full_evals_per_s": _fin(P * 1e3 / t_sobol),
                "sobol_full_ms": _fin(t_sobol),
                "repair_population_ms": _fin(t_repair),
                "mix_class_ms": _fin(t_mix),
                "mix_class_evals_per_s": _fin(P * G * 1e3 / t_mix),
                "mix_class_accept_frac": _fin(mix_accept_frac),
                "samples_per_launch": prof["samples"] / max(prof["launches"], 1),
                "band_entries_per_launch": prof["band_entries"] / max(prof["launches"], 1),
                "partial_fos_sweep": sweep,
                "plain_load_full_evals_per_s": _fin(P * 1e3 / t_plain),
                "plain_load_full_ms": _fin(t_plain),
                "per_gpu_note": "breakdown figures are this rank's (per GPU)",
            },
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
