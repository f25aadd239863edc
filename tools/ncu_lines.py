"""Dev tool: per-source-line instruction and stall shares of one kernel in an ncu report
(all source files of the kernel)."""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
data, fname, cols = [], "?", None
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        cols = (r.index("Warp Stall Sampling (All Samples)"), r.index("Instructions Executed"))
        continue
    if cols and r[0].isdigit():
        num = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
        data.append((fname, int(r[0]), r[1], num(r[cols[0]]), num(r[cols[1]])))
ts = sum(d[3] for d in data) or 1
ti = sum(d[4] for d in data) or 1
print("stall samples", ts, "instructions", ti)
for d in sorted(data, key=lambda d: -d[4])[:top]:
    print("%-14s %5d %5.1f%% %5.1f%%  %s" % (d[0][:14], d[1], 100 * d[3] / ts, 100 * d[4] / ti, d[2].strip()[:90]))
