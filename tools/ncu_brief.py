"""Summarise one kernel of an .ncu-rep: key metrics, stall mix, per-exec-class SASS mix.

usage: python tools/ncu_brief.py REPORT [units_for_class_normalisation]
"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, timeout=600).stdout


want = {"Duration", "Elapsed Cycles", "Registers Per Thread", "Achieved Occupancy", "Executed Ipc Active",
        "Issue Slots Busy", "Executed Instructions", "Theoretical Occupancy", "DRAM Throughput",
        "Memory Throughput", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block"}
for r in csv.reader(io.StringIO(ncu("--page", "details", "--csv"))):
    if len(r) > 14 and r[12] in want:
        print(f"{r[12]:32s} {r[14]:>14s} {r[13]}")
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hdr, rows = rows[1], rows[2:]
ci = hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot_s = sum(int(r[si]) for r in rows)
st = collections.Counter()
for r in rows:
    for c in stall_cols:
        if r[c] not in ("", "0"):
            st[hdr[c]] += int(r[c])
print("stalls:", ", ".join(f"{k[6:]} {100 * v / tot_s:.0f}%" for k, v in st.most_common(8)))
tot = sum(int(r[ci]) for r in rows)
print(f"instructions {tot} = {tot / units:.0f} per unit")
cls = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in rows:
    c = round(int(r[ci]) / units, 1)
    src = r[1].strip()
    op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
    cls[c][0] += 1
    cls[c][1] += int(r[si])
    cls[c][2][op] += 1
for c in sorted(cls, key=lambda c: -c * cls[c][0])[:10]:
    n, s, ops = cls[c]
    print(f"exec/unit {c:5.1f} static {n:4d} -> {c * n:7.0f}/unit  samples {100 * s / tot_s:4.1f}%  "
          + " ".join(f"{o}:{k}" for o, k in ops.most_common(10)))
