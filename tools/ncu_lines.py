"""Dev tool: per-source-line instruction and stall shares of one kernel in an ncu report."""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
h = rows[hdr[0]]
ie = h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
end = hdr[1] if len(hdr) > 1 else len(rows)
data = [(int(r[0]), r[1], int(r[ws] or 0), int(r[ie] or 0))
        for r in rows[hdr[0] + 1:end] if r and r[0].isdigit()]
ts = sum(d[2] for d in data) or 1
ti = sum(d[3] for d in data) or 1
print("stall samples", ts, "instructions", ti)
for d in sorted(data, key=lambda d: -d[3])[:top]:
    print("%5d %5.1f%% %5.1f%%  %s" % (d[0], 100 * d[2] / ts, 100 * d[3] / ti, d[1].strip()[:100]))
