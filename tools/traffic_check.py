"""Cross-check of the ablation kernels' measured traffic against the reference's closed-form traffic
oracle (count_expected_loads, reference oracle.py:72-124; restated in
paper_2002_03258_b200/traffic.py:paper_algorithm_loads) — SURVEY.md §8 row a11.

  python tools/traffic_check.py ncu [m] [n]   # on the GPU box: every case under ncu, one process each
  python tools/traffic_check.py run CASE m n  # one call of CASE (what ncu profiles)

Cases: the paper's V0 (inner product), V1 (outer product, t2 columns per pass), V2 (+ shared B
tile) at t2 = n and t2 < n, and the production V3 kernel. A is m x m fp64 (m = 8192: 537 MB, 4x
the L2), so every pass over A is a DRAM pass and ncu's dram__bytes_read must be ~ eb x loads["A"]
(+ B, C). Global load / store instructions (SASS warp counters x 32 lanes) are compared with the
oracle's per-element load / store totals. Writes profiles/traffic_<tag>.json.
"""

import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {  # name: (variant, t1, t2, t3, impl)
    "v0": ("v0", 128, 1, 1, "ablation"),
    "v1_t2n": ("v1", 128, None, 1, "ablation"),
    "v1_t2_2": ("v1", 128, 2, 1, "ablation"),
    "v2_t2n": ("v2", 128, None, 4, "ablation"),
    "v2_t2_4": ("v2", 128, 4, 4, "ablation"),
    "v3_b200": ("v3", 128, None, 4, "auto"),
}
METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__sass_inst_executed_op_global_ld.sum",
           "smsp__sass_inst_executed_op_global_st.sum", "gpu__time_duration.sum"]


def run_case(name, m, n):
    import torch

    import paper_2002_03258_b200 as tsm
    v, t1, t2, t3, impl = CASES[name]
    t2 = n if t2 is None else t2
    A = tsm.colmajor_empty(m, m, torch.float64, "cuda")
    tsm.fill_uniform(A, seed=1)
    B = tsm.colmajor_empty(m, n, torch.float64, "cuda")
    tsm.fill_uniform(B, seed=2)
    C = tsm.colmajor_empty(m, n, torch.float64, "cuda")
    C.zero_()
    torch.cuda.synchronize()
    p = tsm.KernelParams(t1=t1, t2=t2, t3=t3, variant=tsm.Variant.parse(v))
    tsm.gemm(A, B, C, variant=v, params=p, impl=impl, c_is_zero=True)
    torch.cuda.synchronize()
    ref = (A @ B)
    err = float(((C - ref).norm() / ref.norm()).item())
    assert err < 1e-12, (name, err)


def ncu_case(name, m, n):
    cmd = ["ncu", "--csv", "--metrics", ",".join(METRICS), "-k", "regex:ablation|tsm2r_stream|prep_dyn",
           sys.executable, os.path.abspath(__file__), "run", name, str(m), str(n)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=ROOT)
    rows = list(csv.reader(out.stdout.splitlines()))
    start = next((i for i, r in enumerate(rows) if r and r[0] == "ID"), None)
    if start is None:
        return {"error": (out.stdout + out.stderr)[-2000:]}
    hdr = rows[start]
    ki, ni, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
    tot, kernels = {}, {}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        try:
            val = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        except ValueError:  # "n/a": metric not collected for this kernel
            continue
        tot[r[ni]] = tot.get(r[ni], 0.0) + val
        kernels[r[ki].split("(")[0]] = 1
    tot["kernels"] = sorted(kernels)
    return tot


def expected(name, m, n):
    from paper_2002_03258_b200 import traffic
    v, t1, t2, t3, impl = CASES[name]
    t2 = n if t2 is None else t2
    k = m
    cnt = traffic.paper_algorithm_loads(v, m, k, n, t1, t2, t3)
    loads, stores = dict(cnt["loads"]), dict(cnt["stores"])
    if v in ("v1", "v2"):
        loads["C"] = 0  # zero-C call: V1/V2 start their registers at 0 instead of reading C
    eb = 8
    return {"loads": loads, "stores": stores, "thread_loads_total": sum(loads.values()),
            "thread_stores_total": sum(stores.values()),
            # DRAM: every pass over A misses the L2 (A = 4x L2); B and C are L2-resident
            "dram_read_expected": eb * (loads["A"] + k * n), "a_passes": loads["A"] / (m * k)}


def main():
    mode = sys.argv[1]
    if mode == "run":
        run_case(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
        return
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    tag = os.environ.get("TAG", "r02")
    res = {"what": "ablation kernels' measured traffic vs the reference's count_expected_loads (oracle.py:72-124)",
           "shape": {"m": m, "k": m, "n": n, "precision": "double", "A_bytes": 8 * m * m}, "cases": {}}
    for name in CASES:
        meas = ncu_case(name, m, n)
        exp = expected(name, m, n)
        row = {"expected": exp, "measured": meas}
        if "error" not in meas:
            rd = meas.get("dram__bytes_read.sum", 0.0)
            row["dram_read_ratio"] = round(rd / exp["dram_read_expected"], 4)
            ld = meas.get("smsp__sass_inst_executed_op_global_ld.sum")
            st = meas.get("smsp__sass_inst_executed_op_global_st.sum")
            if ld is not None and CASES[name][4] == "ablation":
                # ncu counts warp instructions; every lane is active (m a multiple of t1 = 128)
                row["thread_loads_ratio"] = round(32 * ld / exp["thread_loads_total"], 4)
                row["thread_stores_ratio"] = round(32 * st / exp["thread_stores_total"], 4) if st is not None else None
        res["cases"][name] = row
        print(json.dumps({name: {k_: v_ for k_, v_ in row.items() if k_ != "expected"}}), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"traffic_{tag}.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
