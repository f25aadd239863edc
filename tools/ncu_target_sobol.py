"""ncu target (dev tool): C4 full evaluation with the Sobol sampler (NEXT-1), twice."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2303_04873_b200 import morea  # noqa: E402
from synth import make_workload  # noqa: E402
w = make_workload(4)
ctx = morea.Context.from_workload(w)
ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
dev = torch.device("cuda:0")
off = torch.from_numpy(w.offsets).to(dev)
obj = torch.empty((w.P, 3), dtype=torch.float64, device=dev)
acc = torch.empty((w.P, 6), dtype=torch.int64, device=dev)
for _ in range(2):
    ctx.eval_full(off, obj, acc, None)
torch.cuda.synchronize()
print("done", obj[1].tolist())
