"""Dev tool: one warm Sobol full evaluation at C4 (for ncu launch lists of library variants)."""
import os, pickle, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_04873_b200 import morea
w, go, ch, nv = pickle.load(open("/tmp/ab_wl4.pkl", "rb"))
ctx = morea.Context.from_workload(w)
ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
dev = torch.device("cuda:0")
off = torch.from_numpy(w.offsets).to(dev); P = w.P
obj = torch.empty((P, 3), dtype=torch.float64, device=dev)
acc = torch.empty((P, 6), dtype=torch.int64, device=dev)
for _ in range(2):
    ctx.eval_full(off, obj, acc, None)
torch.cuda.synchronize()
print("ok")
