import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_04873_b200 import morea
from synth import make_workload
w = make_workload(2)
dev = torch.device("cuda:0")
mode = sys.argv[1]
def make(pairs, no_tex):
    os.environ["MOREA_NO_TEX"] = "1" if no_tex else "0"
    ctx = morea.Context(0)
    sel = pairs
    def sub(off, xyz):
        parts = [xyz[off[i]:off[i+1]] for i in sel]
        o = np.concatenate([[0], np.cumsum([len(p) for p in parts])]).astype(np.int64)
        return o, np.vstack(parts).astype(np.float32)
    cso, csx = sub(w.cs_off, w.cs_xyz); cto, ctx_ = sub(w.ct_off, w.ct_xyz)
    ctx.load_images(w.dims, w.spacing, w.I_s, w.I_t, cso, csx, cto, ctx_, w.r_mm)
    ctx.set_mesh(w.base, w.tets, w.c_delta)
    return ctx
def ev(ctx):
    off = torch.from_numpy(w.offsets[:4]).to(dev)
    acc = torch.empty((4, 6), dtype=torch.int64, device=dev)
    ctx.eval_full(off, None, acc, None)
    torch.cuda.synchronize()
    return morea.acc_to_numpy(acc)["g_sum"]
if mode == "single":
    for nt in (True, False):
        c = make([0], nt); print("pair0 only, notex" if nt else "pair0 only, tex", ev(c)); c.close()
elif mode == "two":
    c1 = make([0, 1, 2, 3], True); g1 = ev(c1); m1 = c1.distance_map(0, 0); c1.close()
    c2 = make([0], True); g2 = ev(c2); m2 = c2.distance_map(0, 0)
    print("all pairs", g1, "\npair0", g2, "\nmap equal", np.array_equal(m1, m2))
    c3 = make([0], True); print("pair0 again", ev(c3))
