"""Summarise ncu outputs into profiles/ (dev tool, runs here without a GPU).

usage: python tools/summarize_ncu.py <round tag> <launches.csv> <prof.ncu-rep> [<prof2.ncu-rep> ...]
Writes profiles/<tag>_launches.txt (per-kernel share of the launch list),
profiles/<tag>_ncu_raster.txt (key metrics of the captured k_raster launches)
and profiles/ncu_summary.json (DRAM bytes per k_raster launch, read by bench.py).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
rep = reps[0]
prof = os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)

rows = list(csv.reader(open(launches)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ik, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
per = {}
seq = []
for r in rows[h + 1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0].replace("morea::", "")
    t = float(r[iv].replace(",", ""))
    per.setdefault(name, []).append(t)
    seq.append((int(r[iid]), name, t))
tot = sum(sum(v) for v in per.values())
out = [f"# ncu launch list ({os.path.basename(launches)}): gpu__time_duration.sum, --clock-control none,",
       "# cold-cache serialised launches of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras`",
       f"# total {tot/1e6:.3f} ms over {len(seq)} launches", "",
       f"{'kernel':28s} {'launches':>8s} {'total ms':>10s} {'mean ms':>9s} {'share':>7s}"]
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    out.append(f"{k:28s} {len(v):8d} {sum(v)/1e6:10.3f} {sum(v)/len(v)/1e6:9.3f} {100*sum(v)/tot:6.1f}%")
load_time = {"k_distance_maps", "k_band_mask", "k_own_records", "k_validate_volume", "k_fill_int", "k_pad_volume", "k_dilate_band"}
step_tot = sum(sum(v) for k, v in per.items() if k not in load_time and not k.startswith("void at::"))
out += ["", "# share of the per-step kernels (load-time and torch fill kernels excluded)"]
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    if k in load_time or k.startswith("void at::"):
        continue
    out.append(f"{k:28s} {100*sum(v)/step_tot:6.1f}%")
out += ["", "# launch sequence (id, kernel, ms)"] + [f"{i:5d} {n:28s} {t/1e6:10.4f}" for i, n, t in seq]
open(os.path.join(prof, f"{tag}_launches.txt"), "w").write("\n".join(out) + "\n")

hdr, units, data = None, None, []
for rp in reps:
    raw = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if hdr is None:
        hdr, units = rr[0], rr[1]
    data += [dict(zip(rr[0], d)) for d in rr[2:]]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
        "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warps_issue_stalled_lg_throttle_per_warp_active.pct",
        "smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warps_issue_stalled_wait_per_warp_active.pct",
        "smsp__warps_issue_stalled_math_pipe_throttle_per_warp_active.pct",
        "smsp__warps_issue_stalled_no_instruction_per_warp_active.pct",
        "smsp__warps_issue_stalled_mio_throttle_per_warp_active.pct",
        "smsp__warps_issue_stalled_tex_throttle_per_warp_active.pct",
        "smsp__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
lines = [f"# ncu --set full of k_raster ({', '.join(os.path.basename(r) for r in reps)}), one row per captured launch", ""]
dram = []
for m in data:
    lines.append(f"launch {m.get('ID')} {m.get('Kernel Name','')[:40]}")
    for k in want:
        if k in m:
            lines.append(f"  {k:70s} {m[k]} {units[hdr.index(k)]}")
    try:
        rb = float(m["dram__bytes_read.sum"].replace(",", ""))
        wb = float(m["dram__bytes_write.sum"].replace(",", ""))
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        sr = sc.get(units[hdr.index("dram__bytes_read.sum")], 1)
        sw = sc.get(units[hdr.index("dram__bytes_write.sum")], 1)
        if rb == rb and wb == wb:  # skip launches ncu could not replay (nan)
            dram.append(rb * sr + wb * sw)
    except Exception:
        pass
    lines.append("")
open(os.path.join(prof, f"{tag}_ncu_raster.txt"), "w").write("\n".join(lines) + "\n")
def _num(m, k):
    try:
        v = float(m[k].replace(",", ""))
        return v if v == v else None
    except Exception:
        return None


rates = {k: [x for x in (_num(m, k) for m in data) if x is not None]
         for k in ("lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
                   "smsp__issue_active.avg.pct_of_peak_sustained_active")}
summ = {"round": tag, "source": [os.path.basename(r) for r in reps],
        "k_raster_dram_bytes_per_launch": (sum(dram) / len(dram)) if dram else None,
        "k_raster_dram_bytes_each": dram,
        "k_raster_l2_hit_pct": rates["lts__t_sector_hit_rate.pct"],
        "k_raster_l1tex_hit_pct": rates["l1tex__t_sector_hit_rate.pct"],
        "k_raster_issue_active_pct": rates["smsp__issue_active.avg.pct_of_peak_sustained_active"]}
json.dump(summ, open(os.path.join(prof, "ncu_summary.json"), "w"), indent=1)
print("\n".join(out[:14]))
print("\n".join(lines[:60]))
