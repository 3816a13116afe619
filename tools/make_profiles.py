"""Summarise ncu output of a bench run into profiles/ (tracked).

    python tools/make_profiles.py ROUND LAUNCHES_CSV FULL_REP [BENCH_JSON]

Writes profiles/<round>_launches.txt (per-kernel launch-list shares),
profiles/<round>_<kernel>_ncu.txt (headline metrics, stall reasons) and
profiles/ncu_summary.json (dram bytes per launch of the dominant kernel, read
by bench.py for roofline.traffic).
"""

import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"
STEP_KERNELS = ("bounds_kernel", "rescore_kernel", "fit_kernel")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
    agg = collections.defaultdict(list)
    for r in data:
        agg[r[ik]].append(float(r[iv].replace(",", "")) * scale[r[iu]])
    return agg


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def main():
    rnd, launch_csv, full_rep = sys.argv[1], sys.argv[2], sys.argv[3]
    bench = json.load(open(sys.argv[4])) if len(sys.argv) > 4 else None
    PROF.mkdir(exist_ok=True)
    agg = launches(launch_csv)
    total = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list ({launch_csv}): gpu__time_duration.sum, --clock-control none",
             "# cold-cache, serialised launches: compare SHARES, not absolute times", ""]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{len(v):6d} launches  {sum(v):12.1f} us total  {sum(v)/len(v):10.2f} us mean  "
                     f"{100*sum(v)/total:5.1f}%  {k}")
    # the throughput step's kernels (bounds_kernel<1, 1> is the zero-copy e2e leg)
    step = {k: v for k, v in agg.items()
            if any(n in k for n in STEP_KERNELS) and "bounds_kernel<1, 1>" not in k}
    if step:
        per = {k: sum(v) / len(v) for k, v in step.items()}
        tot_step = sum(per.values())
        lines += ["", "# shares of one throughput step (mean launch time of each step kernel; the",
                  "# fused strip_kernel launches are the single-frame latency leg, bounds_kernel<1, 1>",
                  "# the zero-copy e2e leg, cnn/select the learned leg)"]
        for k, v in sorted(per.items(), key=lambda kv: -kv[1]):
            lines.append(f"{v:10.2f} us mean  {100 * v / tot_step:5.1f}% of step  {k}")
    (PROF / f"{rnd}_launches.txt").write_text("\n".join(lines) + "\n")

    hdr, units, vals = ncu_raw(full_rep)
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    v0 = vals[0]
    rec = {h: (v0[i], units[i]) for i, h in enumerate(hdr) if h in want}
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v0[i])
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    name = rec.get("Kernel Name", ("kernel", ""))[0]
    out = [f"# ncu --set full --clock-control none capture: {full_rep}", f"kernel: {name}", ""]
    for h in want[1:]:
        if h in rec:
            out.append(f"{h:60s} {rec[h][0]:>16s} {rec[h][1]}")
    out.append("")
    out.append("warp stall samples: " + ", ".join(
        f"{k} {100*v/tot:.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v / tot >= 0.02))
    base = name.split("<")[0].split("(")[0].split()[-1]   # drop "void", template args, params
    short = "strip" if "strip_kernel" in name else base.split("::")[-1]
    (PROF / f"{rnd}_{short}_ncu.txt").write_text("\n".join(out) + "\n")

    def num(h):
        v, u = rec[h]
        x = float(v.replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    summ = {"round": rnd, "kernel": name,
            "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
            "duration_us_ncu": float(rec["gpu__time_duration.sum"][0].replace(",", "")) *
            {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
            [rec["gpu__time_duration.sum"][1]],
            "stall_top": sorted(st, key=lambda k: -st[k])[:5],
            "source": str(full_rep)}
    if bench:
        summ["bench_value"] = bench.get("value")
        summ["bench_roofline"] = bench.get("roofline")
    (PROF / "ncu_summary.json").write_text(json.dumps(summ, indent=1) + "\n")
    print("\n".join(lines[:8]))
    print("\n".join(out))
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
