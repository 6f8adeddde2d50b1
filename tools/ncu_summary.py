#!/usr/bin/env python3
"""Summarise an ncu report (--set full) or a launch-list CSV into profiles/.

  python tools/ncu_summary.py report gpurun_out/prof.ncu-rep profiles/<name>.json
  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "dram__bytes_read.sum.per_second", "l1tex__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    # tcgen05 (k_m2l_i8)
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        ent = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                v = d[k].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                ent[k] = {"value": v, "unit": u.get(k, "")}
        kernels.append(ent)
    return {"source": path, "kernels": kernels}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg, dram = {}, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0]
        val = float(d["Metric Value"].replace(",", ""))
        if d.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            unit = d.get("Metric Unit", "byte")
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1.0)
            dram.setdefault(k, [0.0, 0.0])[0 if "read" in d["Metric Name"] else 1] += val * scale
            continue
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = d.get("Metric Unit", "ns")
        agg.setdefault(k, []).append(val * {"ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9}.get(unit, 1.0))
    tot = sum(sum(v) for v in agg.values())
    ks = sorted(agg.items(), key=lambda x: -sum(x[1]))
    out = []
    for k, v in ks:
        e = {"kernel": k, "launches": len(v), "total_ms": sum(v) / 1e6, "avg_ms": sum(v) / len(v) / 1e6,
             "share": sum(v) / tot}
        if k in dram:
            e["dram_read_gb"], e["dram_write_gb"] = dram[k][0] / 1e9, dram[k][1] / 1e9
        out.append(e)
    return {"source": path, "note": "ncu --metrics gpu__time_duration.sum[,dram__bytes_*] --clock-control none: "
                                    "cold-cache, serialised; totals over all launches of the run", "kernels": out}


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    res = report(src) if kind == "report" else launches(src)
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])
