"""Dev tool: launch list of one device-side optimal-mixing call at C4 (run under ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_04873_b200 import morea
from synth import make_workload, fos_plan, partial_request

w = make_workload(4)
ctx = morea.Context.from_workload(w)
dev = torch.device("cuda:0")
P = w.P
plan = fos_plan(w.tets, w.N)
go, ch, nv = partial_request(w, plan, "class", 0)
G = len(go) - 1
off = torch.from_numpy(w.offsets).to(dev)
obj = torch.empty((P, 3), dtype=torch.float64, device=dev)
acc = torch.empty((P, 6), dtype=torch.int64, device=dev)
tc = torch.empty((P, w.T, 4), dtype=torch.float64, device=dev)
ctx.eval_full(off, obj, acc, tc)
mus, Ls = [], []
for g in range(G):
    X = w.offsets[:, ch[go[g]:go[g + 1]], :].reshape(P, -1).astype(np.float64)
    mus.append(X.mean(0)); Ls.append(np.linalg.cholesky(np.cov(X.T, bias=True) + 1e-4 * np.eye(X.shape[1])).ravel())
mu = torch.from_numpy(np.concatenate(mus)).to(dev); L = torch.from_numpy(np.concatenate(Ls)).to(dev)
cl = torch.zeros(P, dtype=torch.int32, device=dev)
fx = torch.from_numpy(w.fixed_axes.astype("uint8")).to(dev)
flags = torch.zeros((P, G), dtype=torch.uint8, device=dev)
for it in range(2):
    ctx.mix_class(off, acc, obj, tc, go, ch, cl, mu, L, fx, None, 0.0, 1, it, 0, flags)
torch.cuda.synchronize()
print("accepted", flags.float().mean().item())
import time
s = torch.cuda.ExternalStream(ctx.stream_handle)
for reps in (1, 2, 4):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(s)
    for it in range(reps):
        ctx.mix_class(off, acc, obj, tc, go, ch, cl, mu, L, fx, None, 0.0, 1, 10 + it, 0, flags)
    b.record(s)
    torch.cuda.synchronize()
    print("reps", reps, "event ms/call", a.elapsed_time(b) / reps, "wall ms/call", (time.perf_counter() - t0) * 1e3 / reps)
t0 = time.perf_counter()
ctx.eval_partial(off, acc, go, ch, torch.from_numpy(nv).to(dev), tc, torch.empty((P * G, 3), dtype=torch.float64, device=dev), torch.empty((P * G, 6), dtype=torch.int64, device=dev))
torch.cuda.synchronize()
print("partial wall ms", (time.perf_counter() - t0) * 1e3)
