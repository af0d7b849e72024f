"""Summarise ncu captures (details/raw CSV exported on the GPU box) into
profiles/ncu_summary_<tag>.json.

    python tools/summarize_ncu.py <tag> [src dir]

One record per capture file; a capture holding several kernels (e.g. the
humanoid30 part/split launches) gets one sub-record per kernel under
"kernels", keyed "<ID>:<kernel template argument>"."""
import csv
import glob
import json
import os
import re
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
WANT_DETAILS = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Registers Per Thread",
                "Achieved Occupancy", "Achieved Active Warps Per SM", "Executed Ipc Active",
                "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction",
                "Dynamic Shared Memory Per Block", "L2 Hit Rate", "L1/TEX Hit Rate", "Grid Size", "Block Size"]
WANT_RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
            "smsp__sass_inst_executed_op_global_ld.sum", "smsp__sass_inst_executed_op_global_st.sum",
            "lts__t_bytes.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "sm__warps_active.avg.per_cycle_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9,
         "usecond": 1e-6, "msecond": 1e-3, "second": 1}


def kname(full):
    m = re.search(r"<([^>]*)>", full)
    return m.group(1) if m else full.split("(")[0]


def summarise(det):
    rows = list(csv.reader(open(det)))
    if not rows:
        return {}
    h = rows[0]
    iID, iK = h.index("ID"), h.index("Kernel Name")
    iM, iU, iV = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    recs = {}
    for r in rows[1:]:
        key = f"{r[iID]}:{kname(r[iK])}"
        rec = recs.setdefault(key, {})
        if r[iM] in WANT_DETAILS and r[iM] not in rec:
            rec[r[iM]] = f"{r[iV]} {r[iU]}".strip()
    raw = det.replace(".details.csv", ".raw.csv")
    if os.path.exists(raw):
        rr = list(csv.reader(open(raw)))
        hdr, units = rr[0], rr[1]
        for row in rr[2:]:
            key = f"{row[hdr.index('ID')]}:{kname(row[hdr.index('Kernel Name')])}"
            rec = recs.setdefault(key, {})
            d = {k: (u, v) for k, u, v in zip(hdr, units, row)}
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
                            st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = \
                                round(float(v), 3)
                    except ValueError:
                        pass
            rec["stall_cycles_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1]))
            if "dram__bytes_read.sum" in rec and "dram__bytes_write.sum" in rec:
                rec["dram_bytes_per_launch"] = rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
    return recs


out = {}
for det in sorted(glob.glob(os.path.join(src, f"prof_{tag}_*.details.csv"))):
    key = os.path.basename(det)[len(f"prof_{tag}_"):-len(".details.csv")]
    recs = summarise(det)
    if len(recs) == 1:
        k, v = next(iter(recs.items()))
        v["kernel"] = k.split(":", 1)[1]
        out[key] = v
    else:
        out[key] = {"kernels": recs}
os.makedirs("profiles", exist_ok=True)
json.dump(out, open(f"profiles/ncu_summary_{tag}.json", "w"), indent=1)
print(json.dumps(out, indent=1))
