"""Dev tool: fraction of C4 samples whose step is skipped as empty space (full and
class-0 partial evaluation)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_04873_b200 import morea
from synth import make_workload, fos_plan, partial_request
w = make_workload(4)
ctx = morea.Context.from_workload(w)
dev = torch.device("cuda:0")
off = torch.from_numpy(w.offsets).to(dev)
P = w.P
obj = torch.empty((P, 3), dtype=torch.float64, device=dev)
acc = torch.empty((P, 6), dtype=torch.int64, device=dev)
tc = torch.empty((P, w.T, 4), dtype=torch.float64, device=dev)
ctx.prof_enable(True)
ctx.prof_read()
ctx.eval_full(off, obj, acc, tc)
f = ctx.prof_read()
plan = fos_plan(w.tets, w.N)
go, ch, nv = partial_request(w, plan, "class", 0)
G = len(go) - 1
po = torch.empty((P * G, 3), dtype=torch.float64, device=dev)
pa = torch.empty((P * G, 6), dtype=torch.int64, device=dev)
ctx.eval_partial(off, acc, go, ch, torch.from_numpy(nv).to(dev), tc, po, pa)
p = ctx.prof_read()
for name, d in (("full", f), ("partial", p)):
    print(name, "samples", d["samples"], "skipped frac", d["skipped"] / d["samples"], "band/sample",
          d["band_entries"] / d["samples"], "ms", d["ms"])
ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
ctx.eval_full(off, obj, acc, tc)
s = ctx.prof_read()
print("sobol full", "samples", s["samples"], "skipped frac", s["skipped"] / max(s["samples"], 1), "ms", s["ms"])
