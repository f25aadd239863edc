"""Dev tool: key metrics, stall reasons and per-source-line instruction / stall shares of
the captured launches in an ncu report (k_raster).  usage: python tools/ncu_sweep.py report [n_lines]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 35
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr = r[0]
KEYS = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__warps_eligible.avg.per_cycle_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'smsp__sass_inst_executed_op_local_ld.sum', 'launch__registers_per_thread']
for row in r[2:]:
    m = dict(zip(hdr, row))
    print(m['Kernel Name'][:50], m.get('ID'))
    st = []
    for k in hdr:
        if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued'):
            try:
                st.append((float(m[k].replace(',', '')), k))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("  stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.1f}%"
                                   for v, k in sorted(st, reverse=True)[:8]))
    for k in KEYS:
        print("  ", k.ljust(70), m.get(k))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
fname, h = None, None
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
for row in rows:
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
    ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    a = agg[(fname, ln)]
    a[0] += num(row[ie])
    a[1] += num(row[ws])
    a[2] = row[1][:85]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print("per source line (first launch): instruction share, stall share")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k[0][:14]:14s}{k[1]:5d} {100 * v[0] / ti:5.1f}% {100 * v[1] / ts:5.1f}%  {v[2]}")
