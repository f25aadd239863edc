"""Dev tool: A/B timing of libmorea.so variants on the C4 workload (one process per
variant, interleaved rounds).  usage: python tools/ab.py build/var/a.so build/var/b.so ..."""
import os, pickle, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CACHE = "/tmp/ab_wl4.pkl"

CHILD = r'''
import os, pickle, sys, json
sys.path.insert(0, %r)
import torch
from paper_2303_04873_b200 import morea
w, go, ch, nv = pickle.load(open(%r, "rb"))
ctx = morea.Context.from_workload(w)
if os.environ.get("AB_SOBOL"): ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
dev = torch.device("cuda:0")
off = torch.from_numpy(w.offsets).to(dev); P = w.P
obj = torch.empty((P, 3), dtype=torch.float64, device=dev)
acc = torch.empty((P, 6), dtype=torch.int64, device=dev)
tc = torch.empty((P, w.T, 4), dtype=torch.float64, device=dev)
G = len(go) - 1
nvd = torch.from_numpy(nv).to(dev)
pobj = torch.empty((P * G, 3), dtype=torch.float64, device=dev)
pacc = torch.empty((P * G, 6), dtype=torch.int64, device=dev)
s = torch.cuda.ExternalStream(ctx.stream_handle)
def t(fn, reps):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps): fn()
    b.record(s); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
full = t(lambda: ctx.eval_full(off, obj, acc, tc), 3 if os.environ.get("AB_SOBOL") else 5)
part = t(lambda: ctx.eval_partial(off, acc, go, ch, nvd, tc, pobj, pacc), 5)
import hashlib
dig = hashlib.sha1(obj.cpu().numpy().tobytes() + acc.cpu().numpy().tobytes() + pobj.cpu().numpy().tobytes() + pacc.cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps({"full_ms": full, "partial_ms": part, "h0": float(acc[1, 0].item()), "digest": dig}))
'''

def main():
    libs = sys.argv[1:]
    if not os.path.exists(CACHE):
        from synth import make_workload, fos_plan, partial_request
        w = make_workload(4)
        plan = fos_plan(w.tets, w.N)
        go, ch, nv = partial_request(w, plan, "class", 0)
        pickle.dump((w, go, ch, nv), open(CACHE, "wb"))
    rounds = int(os.environ.get("AB_ROUNDS", "2"))
    res = {l: [] for l in libs}
    for r in range(rounds):
        for l in libs:
            env = dict(os.environ, MOREA_LIB=os.path.abspath(l))
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, CACHE)], env=env, capture_output=True, text=True)
            line = [x for x in out.stdout.splitlines() if x.startswith("{")]
            res[l].append(line[-1] if line else out.stderr[-300:])
            print(r, l, res[l][-1], flush=True)

main()
