import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_04873_b200 import morea
from synth import make_workload
w = make_workload(2)
dev = torch.device("cuda:0")
def run(no_tex, pairs=None):
    os.environ["MOREA_NO_TEX"] = "1" if no_tex else "0"
    ctx = morea.Context(0)
    K = len(w.pairs)
    sel = list(range(K)) if pairs is None else pairs
    def sub(off, xyz):
        parts = [xyz[off[i]:off[i+1]] for i in sel]
        o = np.concatenate([[0], np.cumsum([len(p) for p in parts])]).astype(np.int64)
        return o, np.vstack(parts).astype(np.float32)
    cso, csx = sub(w.cs_off, w.cs_xyz); cto, ctx_ = sub(w.ct_off, w.ct_xyz)
    ctx.load_images(w.dims, w.spacing, w.I_s, w.I_t, cso, csx, cto, ctx_, w.r_mm)
    ctx.set_mesh(w.base, w.tets, w.c_delta)
    off = torch.from_numpy(w.offsets[:4]).to(dev)
    acc = torch.empty((4, 6), dtype=torch.int64, device=dev)
    ctx.eval_full(off, None, acc, None)
    torch.cuda.synchronize()
    a = morea.acc_to_numpy(acc)
    return a["h_sum"], a["g_sum"]
for pairs in (None, [0], [1], [2], [3], [1, 0]):
    print(pairs, "notex", run(True, pairs), "tex", run(False, pairs), flush=True)
