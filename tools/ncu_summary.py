"""Summarise ncu captures into profiles/ (run here, on the CPU, over reports pulled back by gpurun).

  python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep=workload_name ... [--launches gpurun_out/launches.csv]

Writes/updates profiles/ncu_summary.json: per workload the dominant kernel's DRAM bytes per launch
(`traffic` in bench.py's roofline), duration, clocks, DRAM/L2/SM throughput, pipe utilisation,
issue-stall mix and SM-active spread; and profiles/launches_<tag>.json from a launch-list CSV.
"""

import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_summary.json")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpc__cycles_elapsed.max.per_second",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_active.min", "sm__cycles_active.avg", "sm__cycles_active.max",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size",
]
# pipe / throughput metrics whose exact names vary between ncu versions and chips: every raw column
# matching one of these patterns is recorded (the DMMA/HMMA tensor subpipes carry the fp64/fp32
# tensor-core load; DRAM throughput is reported as dram__ or gpu__dram_ depending on the version)
PATTERNS = [
    r"^(gpu__)?dram__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^dram__bytes\.sum\.per_second$",
    r"^sm__pipe_tensor_subpipe_(dmma|hmma)_cycles_active\.avg\.pct_of_peak_sustained_(active|elapsed)$",
    r"^sm__pipe_(tensor|fp64|shared)_cycles_active\.avg\.pct_of_peak_sustained_(active|elapsed)$",
    r"^sm__inst_executed_pipe_(fp64|fma|lsu|uniform|tensor).*\.avg\.pct_of_peak_sustained_active$",
    r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld\.sum$",
    r"^l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld\.sum$",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
              "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "nsecond": 1e-9, "Ghz": 1e9, "Mhz": 1e6,
              "hz": 1}


def raw(report):
    if report.endswith(".csv"):  # `ncu -i X --page raw --csv` output saved on the GPU box
        out = open(report).read()
    else:
        out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def value(hdr, units, row, key):
    if key not in hdr:
        return None
    i = hdr.index(key)
    v = row[i].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return v
    return x * UNIT_SCALE.get(units[i], 1)


def summarise(report):
    entries = []
    for hdr, units, row in raw(report):
        e = {"kernel": row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for k in KEYS:
            e[k] = value(hdr, units, row, k)
        for name in hdr:
            if name not in e and any(re.match(p, name) for p in PATTERNS):
                e[name] = value(hdr, units, row, name)
        stalls = {}
        for i, name in enumerate(hdr):
            m = re.match(r"smsp__pcsamp_warps_issue_stalled_([a-z_]+)$", name)
            if m and not name.endswith("_not_issued"):
                try:
                    stalls[m.group(1)] = int(float(row[i].replace(",", "")))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        e["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        rd, wr = e["dram__bytes_read.sum"] or 0, e["dram__bytes_write.sum"] or 0
        e["dram_bytes_per_launch"] = rd + wr
        entries.append(e)
    return entries


def launches(csv_path):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[start + 1:]:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * 1e-3)  # ns -> us
    tot = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "avg_us": round(sum(v) / len(v), 2), "share": round(sum(v) / tot, 4)}
            for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))}


def main():
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    args = sys.argv[1:]
    if "--launches" in args:
        i = args.index("--launches")
        path, tag = args[i + 1], args[i + 2]
        del args[i:i + 3]
        with open(os.path.join(ROOT, "profiles", f"launches_{tag}.json"), "w") as fh:
            json.dump(launches(path), fh, indent=1)
    for spec in args:
        report, workload = spec.split("=")
        ents = summarise(report)
        main_k = max(ents, key=lambda e: e["gpu__time_duration.sum"] or 0)
        main_k["report"] = os.path.basename(report)
        data[workload] = main_k
    with open(OUT, "w") as fh:
        json.dump(data, fh, indent=1)
    print(json.dumps(data, indent=1)[:3000])


if __name__ == "__main__":
    main()
