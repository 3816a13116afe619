"""Summary of an ncu --set full capture of the training step's kernels
(tools/ncu_train.py): per kernel duration, grid, occupancy, issue, DRAM and
tensor sub-pipe activity (the HMMA sub-pipe runs the tcgen05 kind::tf32 MMAs).

    python tools/ncu_train_summary.py REPORT
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}


def get(r, name):
    for h, i in col.items():
        if h == name or h.endswith("." + name) or h.endswith(name):
            try:
                return float(r[i].replace(",", ""))
            except ValueError:
                return r[i]
    return None


print(f"{'kernel':34s} {'us':>7s} {'grid':>5s} {'occ%':>5s} {'issue%':>6s} "
      f"{'hmma%':>6s} {'tensor%':>7s}")
for r in rows[2:]:
    name = r[col["Kernel Name"]][:34]
    dur = get(r, "gpu__time_duration.sum")
    cyc = get(r, "sm__cycles_elapsed.avg")
    hm = get(r, "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg")
    tp = get(r, "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
    occ = get(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    iss = get(r, "sm__inst_issued.avg.pct_of_peak_sustained_active")
    dram = get(r, "dram__bytes.sum.per_second")
    grid = get(r, "launch__grid_size")
    print(f"{name:34s} {dur:7.2f} {int(grid):5d} {occ:5.1f} {iss:6.1f} "
          f"{100 * hm / cyc if hm and cyc else 0:6.1f} {tp:7.2f}")
