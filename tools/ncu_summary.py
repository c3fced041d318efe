"""Summarise ncu reports / launch lists into profiles/ (run in the build container)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "launch__waves_per_multiprocessor": "waves",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefront_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread_inst",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul_thread_inst",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd_thread_inst",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:90]}
        for k, name in KEYS.items():
            if k in hdr:
                d[name] = f"{vals[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(vals[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("void ", "")
                agg[name].append(float(d["Metric Value"]) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0))
    tot = sum(sum(v) for v in agg.values())
    out = [{"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v),
            "share": sum(v) / tot} for k, v in agg.items()]
    return sorted(out, key=lambda d: -d["total_us"])


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    res = raw(path) if mode == "rep" else launches(path)
    if mode == "rep" and len(sys.argv) > 3:  # the problem size the capture ran at (for per-pair counts)
        for d in res:
            d["n"] = int(sys.argv[3])
    print(json.dumps(res, indent=1))
