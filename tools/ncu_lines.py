"""Per-CUDA-source-line totals (instructions executed, stall samples) of one
kernel in an .ncu-rep captured with -lineinfo / --import-source on.
usage: python tools/ncu_lines.py REPORT [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, acc, hdr = "?", {}, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or not r[0]:
        continue
    si, ii = 4, 7
    try:
        s, n = int(r[si]), int(r[ii])
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = acc.setdefault(key, [0, 0, r[1][:90]])
    a[0] += s
    a[1] += n
ts = sum(v[0] for v in acc.values()) or 1
ti = sum(v[1] for v in acc.values()) or 1
print(f"total samples {ts}, instructions {ti}")
for (f, ln), (s, n, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*n/ti:5.1f}% ins  {f}:{ln:<4d} {src}")
