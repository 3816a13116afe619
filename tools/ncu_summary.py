"""Summarise an ncu report: headline metrics, stall reasons, per-region SASS instruction counts."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
items = float(sys.argv[2]) if len(sys.argv) > 2 else 4096
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
raw = list(csv.reader(run("--page", "raw", "--csv").splitlines()))
hdr, vals = raw[0], raw[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']
for h, v in zip(hdr, vals):
    if h in want: print(f"{h:60s} {v}")
st = {h.replace('smsp__pcsamp_warps_issue_stalled_', ''): float(v) for h, v in zip(hdr, vals)
      if 'smsp__pcsamp_warps_issue_stalled' in h and not h.endswith('not_issued') and v.replace('.', '').isdigit()}
tot = sum(st.values())
print("stalls:", ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v / tot > 0.02))
rows = list(csv.reader(run("--page", "source", "--csv", "--print-source", "sass").splitlines()))
h2, data = rows[1], rows[2:]
isrc, iex = h2.index("Source"), h2.index("Instructions Executed")
ex = [float(r[iex] or 0) for r in data]
print(f"SASS {len(data)} instr, {sum(ex)/items:.0f} warp-instr per item")
