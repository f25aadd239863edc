"""ncu target (dev tool): C4 full evaluation (warm-up + 1) then one cached partial colour class."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_04873_b200 import morea
from synth import make_workload, fos_plan, partial_request
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = make_workload(idx)
ctx = morea.Context.from_workload(w)
dev = torch.device("cuda:0")
off = torch.from_numpy(w.offsets).to(dev)
P = w.P
obj = torch.empty((P, 3), dtype=torch.float64, device=dev)
acc = torch.empty((P, 6), dtype=torch.int64, device=dev)
tc = torch.empty((P, w.T, 4), dtype=torch.float64, device=dev)
ctx.eval_full(off, obj, acc, tc)
ctx.eval_full(off, obj, acc, tc)
plan = fos_plan(w.tets, w.N)
go, ch, nv = partial_request(w, plan, "class", 0)
G = len(go) - 1
pobj = torch.empty((P * G, 3), dtype=torch.float64, device=dev)
pacc = torch.empty((P * G, 6), dtype=torch.int64, device=dev)
ctx.eval_partial(off, acc, go, ch, torch.from_numpy(nv).to(dev), tc, pobj, pacc)
torch.cuda.synchronize()
print("done", obj[1].tolist(), pobj[0].tolist())
