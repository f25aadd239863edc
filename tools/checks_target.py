"""Device-checks target (tests/test_gpu_debug_checks.py): every kernel family of the
library on a small workload through the C-ABI with host buffers; prints a digest of
every output.  Run with MOREA_LIB=.../libmorea_debug.so (device-side index and
invariant checks) and with the release library: the digests must be equal.
usage: python tools/checks_target.py [cfg]"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

DIG = {}


def dig(name, *arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    DIG[name] = h.hexdigest()[:16]

from paper_2303_04873_b200 import morea  # noqa: E402
from synth import fos_plan, make_workload, partial_request  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = make_workload(cfg, P=8)
ctx = morea.Context.from_workload(w)
P, T = w.P, w.T
obj = np.zeros((P, 3)); acc = np.zeros(P, morea.ACC_DTYPE); tc = np.zeros((P, T, 4))
ctx.eval_full(w.offsets, obj, acc, tc)                                    # k_setup, k_raster, k_reduce
dig("full", obj, acc, tc)
plan = fos_plan(w.tets, w.N)
go, ch, nv = partial_request(w, plan, "class", 0)
G = len(go) - 1
pobj = np.zeros((P * G, 3)); pacc = np.zeros(P * G, morea.ACC_DTYPE)
ctx.eval_partial(w.offsets, acc, go, ch, nv, tc, pobj, pacc)              # cached partial
dig("partial", pobj, pacc)
ctx.eval_partial(w.offsets, acc, go, ch, nv, None, pobj, pacc)            # stateless partial
dig("partial_nocache", pobj, pacc)
cnt = np.zeros(P, np.int32); sev = np.zeros(P); fl = np.zeros((P, 2, T), np.uint8)
ctx.check_folds(w.offsets, cnt, sev, fl)                                  # k_check_folds
dig("folds", cnt, sev, fl)
dig("owner", ctx.owner_map(w.offsets[1], 0))                              # k_owner_map
dig("sample_map", *ctx.sample_map(w.offsets[1], 1))                       # k_raster dump
ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
ctx.eval_full(w.offsets, obj, acc, tc)                                    # k_sobol
dig("sobol_full", obj, acc)
ctx.eval_partial(w.offsets, acc, go, ch, nv, tc, pobj, pacc)
dig("sobol_partial", pobj, pacc)
ctx.set_sampler(morea.SAMPLER_VOXEL)
ctx.eval_full(w.offsets, obj, acc, tc)
off = w.offsets.copy()
ctx.repair(off, 7, w.fixed_axes.astype(np.uint8))                         # k_repair
dig("repair", off)
masks = (w.I_s > 0.25).astype(np.uint8)
dig("labels", ctx.label_counts(None, 0, masks, 1))                        # exports
dig("dvf", *ctx.dvf(w.offsets[1], 0))
d = 6 * (go[1] - go[0])
mu = np.concatenate([w.offsets[:, ch[go[g]:go[g + 1]], :].reshape(P, -1).mean(0) for g in range(G)])
Ls = np.concatenate([(0.05 * np.eye(6 * (go[g + 1] - go[g]))).ravel() for g in range(G)])
ctx.mix_class(off, acc, obj, tc, go, ch, np.zeros(P, np.int32), mu, Ls, w.fixed_axes.astype(np.uint8))
dig("mix", off, obj, acc, tc)
ctx.close()
print(json.dumps(DIG))
print("checks target ok")
