"""Print the key ncu metrics + stall breakdown + top source lines of a report (dev tool)."""
import csv, subprocess, sys
rep = sys.argv[1]
nsamp = float(sys.argv[2]) if len(sys.argv) > 2 else 6.44e9
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines())); hdr, units, d = r[0], r[1], r[2]
m = dict(zip(hdr, d))
rows = []
for k in hdr:
    if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued'):
        try: rows.append((float(m[k].replace(',', '')), k))
        except: pass
tot = sum(v for v, k in rows)
for v, k in sorted(rows, reverse=True)[:8]: print(f'{100*v/tot:5.1f}%  {k.replace("smsp__pcsamp_warps_issue_stalled_","")}')
for k in ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
          'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__warps_eligible.avg.per_cycle_active',
          'l1tex__throughput.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed',
          'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
          'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'l1tex__t_output_wavefronts_pipe_lsu_mem_local_op_ld.sum',
          'launch__registers_per_thread', 'dram__bytes_read.sum', 'lts__t_sector_hit_rate.pct']:
    print(k.ljust(75), m.get(k))
print('warp-inst per 32-sample step', float(m['smsp__inst_executed.sum'].replace(',', '')) / (nsamp / 32))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = next(r for r in rows if r and r[0] == 'Line No')
ie = hdr.index('Instructions Executed')
lines = {}; fname = None
def num(x):
    try: return int(x)
    except: return 0
for r in rows:
    if r and r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if not r or r[0] in ('', 'Line No', 'Function Name'): continue
    try: ln = int(r[0])
    except: continue
    key = (fname, ln)
    if key not in lines: lines[key] = [r[1][:90], 0, 0]
    lines[key][1] += num(r[4]); lines[key][2] += num(r[ie])
tot_s = sum(v[1] for v in lines.values()); tot_i = sum(v[2] for v in lines.values())
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
for k, v in sorted(lines.items(), key=lambda kv: -kv[1][1])[:n]:
    print(f"{k[0][:10]:10s}{k[1]:5d} inst {100*v[2]/tot_i:5.1f}%  stall {100*v[1]/tot_s:5.1f}%  {v[0]}")
