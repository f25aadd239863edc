#!/usr/bin/env python
"""bench.py -- the MOREA hot path on B200 (contract in DESIGN.md §6).

Workload (BASELINE.json configs[3], the paper-scale case that fits one GPU):
C4 = 256x256x96 CT-shaped phantom at 1.5 mm, 600-point Delaunay dual-dynamic
mesh (3607 tets), 7 contour pairs, P = 512 solutions per GPU (weak scaling:
N GPUs evaluate N*512 solutions, the C5 configuration at N = 8).

One step = one MO-RV-GOMEA generation's evaluation work (§4.2.1
L401-410: partial evaluations run one colour class after another):
  full evaluation of the P solutions (writes the per-tet cache),
  a partial evaluation of EVERY FOS colour class in turn (each edge = one
  group, delta on its dependent tets, old contributions from the cache), for
  all P solutions,
  the fold check of the P solutions, and (N > 1) the all-gather of the
  per-solution outputs.
Units per step = P full + P * (sum of the classes' groups) partial evaluations;
the full and partial rates are reported separately next to the blend.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--dist-backend nccl|gloo] [--dump-records PATH]
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


def workload_config(P_total, n_groups, n_classes, world, T, backend):
    return {
        "workload": f"C4 paper-scale: 256x256x96 CT-shaped phantom (1.5 mm), 600-point Delaunay dual mesh "
                    f"({T} tets), 7 contour pairs, P={P_total // world}/GPU (P_total={P_total}); step = one generation: "
                    f"full eval + partial eval of every FOS colour class ({n_classes} classes, {n_groups} "
                    f"edge groups, tet cache) + fold check"
                    + (f" + {backend} all-gather" if world > 1 else ""),
        "population_per_gpu": P_total // world,
        "population_total": P_total,
        "colour_classes": n_classes,
        "partial_groups_per_step": n_groups,
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


def _oracle_solution(w, classes, sol, core, conn):
    """Child process: pinned to one core, 1 full + every class's partial evaluations of one
    solution (the GPU step's full:partial mix); sends (units, seconds)."""
    try:
        os.sched_setaffinity(0, {core})
    except Exception:
        pass
    from oracle.oracle import Oracle
    orc = Oracle.from_workload(w)
    orc.eval(w.offsets[0])  # untimed: the oracle's lazy distance-map memo (load-time work)
    t0 = time.perf_counter()
    _, base = orc.eval(w.offsets[sol])
    units = 1
    for go, ch, nv in classes:
        for g in range(len(go) - 1):
            orc.eval_partial(w.offsets[sol], base, ch[go[g]:go[g + 1]], nv[sol, go[g]:go[g + 1]])
            units += 1
    conn.send((units, time.perf_counter() - t0))
    conn.close()


def oracle_baseline(w, classes, n_proc):
    """The oracle as it stands, per process one solution (1 full + all class partials),
    each process pinned to its own core; n_proc processes on disjoint solutions."""
    import multiprocessing as mproc
    ctx = mproc.get_context("fork")
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count()))
    n_proc = max(1, min(n_proc, len(cores)))
    pipes, procs = [], []
    t0 = time.perf_counter()
    for i in range(n_proc):
        r, s_ = ctx.Pipe(duplex=False)
        pr = ctx.Process(target=_oracle_solution, args=(w, classes, 1 + i, cores[i], s_))
        pr.start()
        pipes.append(r)
        procs.append(pr)
    res = [r.recv() for r in pipes]
    for pr in procs:
        pr.join()
    wall = time.perf_counter() - t0
    units = sum(u for u, _ in res)
    # throughput over the processes' own timed regions (the memo warm-up excluded)
    busy = max(t for _, t in res)
    return units / busy, units, busy, n_proc, wall


def run_reference(args, rank, world):
    """--impl reference: the oracle (plain single-thread C, fp64/int128) on this workload."""
    if rank != 0:
        return 0
    from synth import fos_plan, make_workload, partial_request
    w = make_workload(CONFIG_INDEX, P=P_PER_GPU)
    plan = fos_plan(w.tets, w.N)
    classes = [partial_request(w, plan, "class", c) for c in range(len(plan["classes"]))]
    from oracle.oracle import Oracle
    orc = Oracle.from_workload(w)
    orc.eval(w.offsets[0])
    # each step: a bounded sample of the generation workload: 1 full evaluation and
    # one class's partial evaluations (classes in turn), of one solution
    times, units = [], 0
    for it in range(args.warmup + args.steps):
        sol = 1 + it % (w.P - 1)
        go, ch, nv = classes[it % len(classes)]
        t0 = time.perf_counter()
        _, base = orc.eval(w.offsets[sol])
        for g in range(len(go) - 1):
            orc.eval_partial(w.offsets[sol], base, ch[go[g]:go[g + 1]], nv[sol, go[g]:go[g + 1]])
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
            units += len(go)
    total = sum(times)
    value = units / total
    G = sum(len(c[0]) - 1 for c in classes)
    sample = ("per step: 1 full + the partial evaluations of one FOS colour class (classes in turn) "
              "of one C4 solution, oracle single-threaded")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(P_PER_GPU * world, G, len(classes), world, w.T, "none"),
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
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: records staged through host memory (several ranks may share one GPU)")
    ap.add_argument("--dump-records", default=None, help="rank 0 writes the gathered records (.npy)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-procs", type=int, default=32, help="processes of the oracle x nproc leg (cap)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the Sobol / repair / mixing / plain-load breakdown timings")
    ap.add_argument("--quick", action="store_true",
                    help="timed region only (no breakdown, sweep, e2e or CPU legs): multi-rank checks")
    ap.add_argument("--pop-per-rank", type=int, default=P_PER_GPU,
                    help="solutions per rank (default 512: the C4 / C5 workload)")
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

    dev_index = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    backend = args.dist_backend
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    from paper_2303_04873_b200 import morea
    from paper_2303_04873_b200.distributed import all_gather_records, pack, shard_bounds
    from synth import fos_plan, make_workload, partial_request

    P_total = args.pop_per_rank * world
    w = make_workload(CONFIG_INDEX, P=P_total)
    plan = fos_plan(w.tets, w.N)
    classes = [partial_request(w, plan, "class", c) for c in range(len(plan["classes"]))]
    n_cls = len(classes)
    Gs = [len(c[0]) - 1 for c in classes]
    G_tot = sum(Gs)
    s0, s1 = shard_bounds(P_total, world, rank)
    P = s1 - s0

    ctx = morea.Context.from_workload(w, device=dev_index)
    stream = torch.cuda.ExternalStream(ctx.stream_handle, device=dev)
    T = w.T
    for go, ch, _ in classes:  # build every class's dependent-tet plan up front (cached)
        ctx.prepare_partial(go, ch)
    off_d = torch.from_numpy(w.offsets[s0:s1].copy()).to(dev)
    nv_d = [torch.from_numpy(c[2][s0:s1].copy()).to(dev) for c in classes]
    obj_d = torch.empty((P, 3), dtype=torch.float64, device=dev)
    acc_d = torch.empty((P, 6), dtype=torch.int64, device=dev)
    cache_d = torch.empty((P, T, 4), dtype=torch.float64, device=dev)
    pobj_d = [torch.empty((P * G, 3), dtype=torch.float64, device=dev) for G in Gs]
    pacc_d = [torch.empty((P * G, 6), dtype=torch.int64, device=dev) for G in Gs]
    cnt_d = torch.empty(P, dtype=torch.int32, device=dev)
    sev_d = torch.empty(P, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def gather():
        outs = []
        with torch.cuda.stream(stream):
            outs.append(all_gather_records(pack(obj_d, acc_d), P_total))
            for c in range(n_cls):
                outs.append(all_gather_records(pack(pobj_d[c], pacc_d[c]), P_total, rows_per_solution=Gs[c]))
        return outs

    def partials():
        for c, (go, ch, _) in enumerate(classes):
            ctx.eval_partial(off_d, acc_d, go, ch, nv_d[c], cache_d, pobj_d[c], pacc_d[c])

    def step():
        ctx.eval_full(off_d, obj_d, acc_d, cache_d)
        partials()
        ctx.check_folds(off_d, cnt_d, sev_d, None)
        if world > 1:
            return gather()
        return None

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
    with ClockSampler(dev_index) as clk:
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

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_max = max_over_ranks(sum(times))
    units = (P_total + P_total * G_tot) * args.steps
    value = units / (t_max / 1e3)

    if args.dump_records:
        recs = gather() if world > 1 else [pack(obj_d, acc_d)] + [pack(pobj_d[c], pacc_d[c]) for c in range(n_cls)]
        if rank == 0:
            import numpy as _np
            _np.save(args.dump_records, torch.cat([r.cpu() for r in recs]).numpy())

    if args.quick:
        if rank == 0:
            print(json.dumps({
                "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": workload_config(P_total, G_tot, n_cls, world, T, backend),
                "gpu_launches": int(launches), "clocks": clk.summary(), "quick": True}), flush=True)
        ctx.close()
        if world > 1:
            dist.destroy_process_group()
        return 0

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

    peak, peak_src = measured_hbm_peak()

    def prof_run(fn, reps=3):
        """k_raster algorithmic GB/s of fn from the kernel's own counters and CUDA events."""
        fn()
        torch.cuda.synchronize()
        ctx.prof_enable(True)
        ctx.prof_read()
        t = timed(fn, reps)
        sp = ctx.prof_read()
        ctx.prof_enable(False)
        sb = 8 * sp["samples"] + 12 * sp["band_entries"] + 32 * sp["items"]
        gbs = sb / (sp["ms"] / 1e3) / 1e9 if sp["ms"] > 0 else None
        return t, sp, gbs

    # separate full / partial throughputs (same inputs, device time)
    t_full, sp_full, gbs_full = prof_run(lambda: ctx.eval_full(off_d, obj_d, acc_d, cache_d))
    t_parts, sp_parts, gbs_parts = prof_run(partials)
    per_class = []
    for c, (go, ch, _) in enumerate(classes):
        run = (lambda c=c, go=go, ch=ch: ctx.eval_partial(off_d, acc_d, go, ch, nv_d[c], cache_d, pobj_d[c],
                                                          pacc_d[c]))
        t_c, sp_c, gbs_c = prof_run(run)
        per_class.append({"class": c, "groups": Gs[c], "evals_per_s": P * Gs[c] * 1e3 / t_c, "ms": t_c,
                          "k_raster_frac": (gbs_c / peak) if gbs_c else None})
    t_part_nc = timed(lambda: ctx.eval_partial(off_d, acc_d, classes[0][0], classes[0][1], nv_d[0], None,
                                               pobj_d[0], pacc_d[0]))
    # partial-evaluation sweep over FOS sizes: 1 edge, 4 and 16 edges of
    # colour class 0, the whole class as one group, all points as one group; cached
    sweep = {}
    for kind in ("class", "edges4", "edges16", "wholeclass", "all"):
        sgo, sch, snv = partial_request(w, plan, kind, 0)
        sG = len(sgo) - 1
        snv_d = torch.from_numpy(snv[s0:s1].copy()).to(dev)
        spo = torch.empty((P * sG, 3), dtype=torch.float64, device=dev)
        spa = torch.empty((P * sG, 6), dtype=torch.int64, device=dev)
        run = (lambda sgo=sgo, sch=sch, snv_d=snv_d, spo=spo, spa=spa:
               ctx.eval_partial(off_d, acc_d, sgo, sch, snv_d, cache_d, spo, spa))
        t_k, sp, gbs = prof_run(run)
        sweep[kind] = {"groups": sG, "points_per_group": round(len(sch) / sG, 2),
                       "evals_per_s": P * sG * 1e3 / t_k, "ms": t_k,
                       "k_raster_gbs": gbs, "k_raster_frac": (gbs / peak) if gbs else None,
                       "samples_per_eval": sp["samples"] / max(sp["launches"], 1) / (P * sG)}
    t_sobol = t_repair = t_mix = t_plain = float("nan")
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
        go0, ch0, _ = classes[0]
        offs_h = w.offsets[s0:s1]
        mus, Ls = [], []
        for g in range(Gs[0]):
            X = offs_h[:, ch0[go0[g]:go0[g + 1]], :].reshape(offs_h.shape[0], -1).astype(_np.float64)
            C = _np.cov(X.T, bias=True) + 1e-4 * _np.eye(X.shape[1])
            mus.append(X.mean(0))
            Ls.append(_np.linalg.cholesky(C).ravel())
        mu_d = torch.from_numpy(_np.concatenate(mus)).to(dev)
        L_d = torch.from_numpy(_np.concatenate(Ls)).to(dev)
        cl_d = torch.zeros(P, dtype=torch.int32, device=dev)
        ctx.eval_full(off_d, obj_d, acc_d, cache_d)  # voxel-mode state of off_d (the Sobol run overwrote it)
        mx_off, mx_acc, mx_obj, mx_tc = off_d.clone(), acc_d.clone(), obj_d.clone(), cache_d.clone()
        mx_flags = torch.zeros((P, Gs[0]), dtype=torch.uint8, device=dev)

        def mix_once():
            mx_off.copy_(off_d); mx_acc.copy_(acc_d); mx_obj.copy_(obj_d); mx_tc.copy_(cache_d)
            ctx.mix_class(mx_off, mx_acc, mx_obj, mx_tc, go0, ch0, cl_d, mu_d, L_d, fixed_d, None, 0.0, 2024, 0,
                          s0, mx_flags)
        mix_once()  # first call allocates the mixing scratch
        t_mix = timed(mix_once, reps=2)
        mix_accept_frac = float(mx_flags.float().mean().item())
        # plain-load path (volumes beyond the 2D gather-texture limits): MOREA_NO_TEX context
        os.environ["MOREA_NO_TEX"] = "1"
        ctx_plain = morea.Context.from_workload(w, device=dev_index)
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
        ctx.eval_full(off_d, obj_d, acc_d, cache_d)

    # ---- roofline of the dominant kernel (k_raster), SURVEY.md §8(d) algorithmic bytes
    alg_bytes = 8 * prof["samples"] + 12 * prof["band_entries"] + 32 * prof["items"]
    achieved = alg_bytes / (prof["ms"] / 1e3) / 1e9 if prof["ms"] > 0 else None
    per_launch_bytes = alg_bytes / max(prof["launches"], 1)
    ncu = ncu_summary()
    traffic = ncu.get("k_raster_dram_bytes_per_launch")

    # ---- e2e: the same step through the public API, inputs copied from pinned host memory
    # and the results read back to pinned host memory inside the timed region
    off_h = torch.from_numpy(w.offsets[s0:s1].copy()).pin_memory()
    nv_h = [torch.from_numpy(c[2][s0:s1].copy()).pin_memory() for c in classes]
    obj_h = torch.empty((P, 3), dtype=torch.float64).pin_memory()
    acc_h = torch.empty((P, 6), dtype=torch.int64).pin_memory()
    pobj_h = [torch.empty((P * G, 3), dtype=torch.float64).pin_memory() for G in Gs]
    pacc_h = [torch.empty((P * G, 6), dtype=torch.int64).pin_memory() for G in Gs]
    cnt_h = torch.empty(P, dtype=torch.int32).pin_memory()
    sev_h = torch.empty(P, dtype=torch.float64).pin_memory()

    # (copies on torch's default stream: the legacy default stream orders them
    # against the context stream, which is a blocking stream, both ways)
    def step_e2e():
        off_d.copy_(off_h, non_blocking=True)
        for c in range(n_cls):
            nv_d[c].copy_(nv_h[c], non_blocking=True)
        step()
        obj_h.copy_(obj_d, non_blocking=True)
        acc_h.copy_(acc_d, non_blocking=True)
        for c in range(n_cls):
            pobj_h[c].copy_(pobj_d[c], non_blocking=True)
            pacc_h[c].copy_(pacc_d[c], non_blocking=True)
        cnt_h.copy_(cnt_d, non_blocking=True)
        sev_h.copy_(sev_d, non_blocking=True)
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
    e2e_value = units / max_over_ranks(sum(e2e_times))
    h2d = off_h.numel() * 4 + sum(x.numel() * 4 for x in nv_h)
    d2h = (obj_h.numel() + acc_h.numel() + sum(x.numel() for x in pobj_h) + sum(x.numel() for x in pacc_h)) * 8 \
        + cnt_h.numel() * 4 + sev_h.numel() * 8

    # ---- CPU baseline: the oracle as it stands (rank 0, N = 1 only): one solution's
    # generation work (1 full + every class's partials) on one pinned core, and the same
    # per process on min(nproc, --cpu-procs) cores (disjoint solutions)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v1, u1, t1, _, _ = oracle_baseline(w, classes, 1)
        vn, un, tn, npr, wall = oracle_baseline(w, classes, args.cpu_procs)
        cpu = {"value": v1, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"one C4 solution's generation work: 1 full + {u1 - 1} partial evaluations (every "
                         f"1-edge group of all {n_cls} FOS colour classes, the GPU step's mix), one process "
                         f"pinned to one core (sched_setaffinity), {t1:.1f} s",
               "oracle_x_nproc": {"value": vn, "processes": npr, "units": un, "seconds": tn,
                                  "note": "one solution per process, each pinned to its own core; "
                                          "throughput over the slowest process's timed region"},
               **host_cpu()}

    if rank == 0:
        full_rate = P_total * 1e3 / t_full
        part_rate = P_total * G_tot * 1e3 / t_parts
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "value_full_evals_per_s": full_rate,
            "value_partial_evals_per_s": part_rate,
            "config": workload_config(P_total, G_tot, n_cls, world, T, backend),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": traffic, "kernel": "k_raster",
                         "frac_full_launch": (gbs_full / peak) if gbs_full else None,
                         "frac_partial_launches": (gbs_parts / peak) if gbs_parts else None,
                         "algorithmic_bytes_per_launch": per_launch_bytes, "peak_source": peak_src,
                         "launches": prof["launches"], "kernel_ms": prof["ms"],
                         "ncu": {"source": ncu.get("source"), "l2_hit_pct": ncu.get("k_raster_l2_hit_pct"),
                                 "l1tex_hit_pct": ncu.get("k_raster_l1tex_hit_pct"),
                                 "issue_active_pct": ncu.get("k_raster_issue_active_pct")}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "breakdown": {
                "full_evals_per_s": full_rate / world, "full_ms": t_full,
                "partial_evals_per_s_all_classes": part_rate / world, "partial_ms_all_classes": t_parts,
                "partial_per_class": per_class,
                "partial_class0_nocache_evals_per_s": P * Gs[0] * 1e3 / t_part_nc,
                "sobol_full_evals_per_s": _fin(P * 1e3 / t_sobol),
                "sobol_full_ms": _fin(t_sobol),
                "repair_population_ms": _fin(t_repair),
                "mix_class_ms": _fin(t_mix),
                "mix_class_evals_per_s": _fin(P * Gs[0] * 1e3 / t_mix),
                "mix_class_accept_frac": _fin(mix_accept_frac),
                "samples_per_launch": prof["samples"] / max(prof["launches"], 1),
                "quiet_row_sample_frac": (prof["skipped"] / prof["samples"]) if prof["samples"] else None,
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
    rc = main()
    # leave without the interpreter's teardown of CUDA-owning objects (torch tensors
    # freed after the context stream is gone); everything is flushed and finished here
    sys.stdout.flush()
    sys.stderr.flush()
    os._exit(rc)
