"""Summarise ncu captures (details/raw CSV exported on the GPU box) into
profiles/ncu_summary_<tag>.json."""
import csv
import glob
import json
import os
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
WANT_DETAILS = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Registers Per Thread",
                "Achieved Occupancy", "Achieved Active Warps Per SM", "Executed Ipc Active",
                "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction",
                "Dynamic Shared Memory Per Block", "L2 Hit Rate", "L1/TEX Hit Rate"]
WANT_RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
            "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9,
         "usecond": 1e-6, "msecond": 1e-3, "second": 1}
out = {}
for det in sorted(glob.glob(os.path.join(src, f"prof_{tag}_*.details.csv"))):
    key = os.path.basename(det)[len(f"prof_{tag}_"):-len(".details.csv")]
    rows = list(csv.reader(open(det)))
    h = rows[0]
    iM, iU, iV = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    rec = {}
    for r in rows[1:]:
        if r[iM] in WANT_DETAILS and r[iM] not in rec:
            rec[r[iM]] = f"{r[iV]} {r[iU]}".strip()
    raw = det.replace(".details.csv", ".raw.csv")
    if os.path.exists(raw):
        rr = list(csv.reader(open(raw)))
        d = {k: (u, v) for k, u, v in zip(rr[0], rr[1], rr[2])}
        for k in WANT_RAW:
            if k in d:
                u, v = d[k]
                try:
                    val = float(v.replace(",", ""))
                    rec[k] = val * SCALE[u] if u in SCALE else val
                except ValueError:
                    rec[k] = v
        st = {}
        for k, (u, v) in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    if float(v) >= 0.05:
                        st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
                except ValueError:
                    pass
        rec["stall_cycles_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1]))
        if "dram__bytes_read.sum" in rec and "dram__bytes_write.sum" in rec:
            rec["dram_bytes_per_launch"] = rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
    out[key] = rec
os.makedirs("profiles", exist_ok=True)
json.dump(out, open(f"profiles/ncu_summary_{tag}.json", "w"), indent=1)
print(json.dumps(out, indent=1))
