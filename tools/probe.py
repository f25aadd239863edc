"""Quick perf probe (dev tool): times full and partial evaluation at C4 with CUDA events."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_04873_b200 import morea
from synth import make_workload, fos_plan, partial_request

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
t0 = time.time(); w = make_workload(idx); print("gen", time.time() - t0, flush=True)
t0 = time.time(); ctx = morea.Context.from_workload(w)
if "sobol" in sys.argv: ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
torch.cuda.synchronize(); print("load", time.time() - t0, flush=True)
dev = torch.device("cuda:0")
off = torch.from_numpy(w.offsets).to(dev)
P = w.P
obj = torch.empty((P, 3), dtype=torch.float64, device=dev)
acc = torch.empty((P, 6), dtype=torch.int64, device=dev)
tc = torch.empty((P, w.T, 4), dtype=torch.float64, device=dev)
s = torch.cuda.ExternalStream(ctx.stream_handle)
ctx.prof_enable(True)
for it in range(3):
    ctx.eval_full(off, obj, acc, tc)
torch.cuda.synchronize()
print("warm", ctx.prof_read(), flush=True)
for it in range(3):
    ctx.eval_full(off, obj, acc, tc)
r = ctx.prof_read(); print("full", r, "evals/s %.1f" % (P * r["launches"] / (r["ms"] / 1e3)), "samples/s %.3g" % (r["samples"] / (r["ms"] / 1e3)), flush=True)
a = morea.acc_to_numpy(acc)
print("n_samples[0:4]", a["n_samples"][:4], "2V", 2 * w.V, "obj0", obj[0].tolist(), "obj1", obj[1].tolist())
plan = fos_plan(w.tets, w.N)
for kind in (("class",) if "quick" in sys.argv else ("class", "edges4", "edges16", "all")):
    go, ch, nv = partial_request(w, plan, kind, 0)
    G = len(go) - 1
    nvd = torch.from_numpy(nv).to(dev)
    pobj = torch.empty((P * G, 3), dtype=torch.float64, device=dev)
    pacc = torch.empty((P * G, 6), dtype=torch.int64, device=dev)
    for cache in (tc, None):
        ctx.eval_partial(off, acc, go, ch, nvd, cache, pobj, pacc)
        torch.cuda.synchronize(); ctx.prof_read()
        for it in range(3):
            ctx.eval_partial(off, acc, go, ch, nvd, cache, pobj, pacc)
        r = ctx.prof_read()
        print(kind, "G", G, "cache" if cache is not None else "nocache", r, "partial evals/s %.3g" % (P * G * r["launches"] / (r["ms"] / 1e3)), "samples/s %.3g" % (r["samples"] / (r["ms"] / 1e3)), flush=True)
