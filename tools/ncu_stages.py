"""Dev tool: instruction and stall-sample shares of one captured k_raster launch, per
function and per stage (row stage / sweep loop / per-sample path / guidance), from the
ncu source page.  usage: python tools/ncu_stages.py report.ncu-rep [launch index]"""
import collections
import csv
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
fname = h = None
agg = collections.defaultdict(lambda: [0.0, 0.0])
text = {}  # source text of morea_kernels.cu as imported into the report (--import-source on)
for row in csv.reader(src.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        h = row
        continue
    try:
        ln = int(row[0])
    except ValueError:
        continue
    if fname == "morea_kernels.cu" and len(row) > 1:
        text.setdefault(ln, row[1])
    ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")

    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    agg[(fname, ln)][0] += num(row[ie])
    agg[(fname, ln)][1] += num(row[ws])

full = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda",
                       "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
fname = None
for row in csv.reader(full.splitlines()):
    if len(row) >= 2 and row[0] in ("File Name", "File Path"):
        fname = row[1].split("/")[-1]
        continue
    if fname == "morea_kernels.cu" and len(row) >= 2:
        try:
            text[int(row[0])] = row[1]
        except ValueError:
            pass
n_lines = max(text) if text else 0
lines = [text.get(i + 1, "") for i in range(n_lines)]
if not any(lines):  # report without imported source: fall back to the working tree
    lines = open(os.path.join(ROOT, "paper_2303_04873_b200/csrc/morea_kernels.cu")).read().split("\n")
starts = []
for i, l in enumerate(lines):
    m = re.match(r"^(?:template.*)?\s*(?:__device__|__global__|static|inline|struct)[^;]*?\b(\w+)\s*\(", l) or \
        re.match(r"^\s{0,2}(?:__device__ __forceinline__|__device__)\s+[\w:<>&\* ]+?\b(\w+)\s*\(", l)
    if m:
        starts.append((i + 1, m.group(1)))


def fn(ln):
    best = "?"
    for s, n in starts:
        if s <= ln:
            best = n
    return best


def find(pat):
    return next(i + 1 for i, l in enumerate(lines) if pat in l)


sweep_start = find("// Sweep in windows")
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
byf = collections.defaultdict(lambda: [0.0, 0.0])
cat = collections.defaultdict(lambda: [0.0, 0.0])
for (f, ln), v in agg.items():
    n = fn(ln) if f == "morea_kernels.cu" else f
    byf[n][0] += v[0]
    byf[n][1] += v[1]
    if n in ("row_interval", "row_interval_exact", "row_interval_exact_if", "slice_y_range", "warp_incl_scan",
             "count_only", "quiet_hull", "quiet_off", "count_quiet"):
        c = "row stage"
    elif n == "raster":
        c = "row stage" if ln < sweep_start else "sweep loop"
    elif n in ("sample", "plerp", "gather_tex", "tri", "exact_fg", "exact_fg_if", "gather"):
        c = "per-sample path"
    elif n in ("entry", "enqueue", "drain"):
        c = "guidance"
    else:
        c = "other: " + n
    cat[c][0] += v[0]
    cat[c][1] += v[1]
print(f"# launch {skip}: {ti:.4g} warp-instructions")
print("per function (instructions, stall samples):")
for k, v in sorted(byf.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {k:32s} {100 * v[0] / ti:5.1f}%  {100 * v[1] / ts:5.1f}%")
print("per stage:")
for k, v in sorted(cat.items(), key=lambda kv: -kv[1][1]):
    if v[0] / ti > 0.004 or v[1] / ts > 0.004:
        print(f"  {k:32s} {100 * v[0] / ti:5.1f}%  {100 * v[1] / ts:5.1f}%")
