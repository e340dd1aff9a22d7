"""Sustained A/B of build-time kernel geometry selected through the environment (TSM2X_RPT,
TSM2X_CW, TSM2X_CONSUMER): each candidate runs in its own process (the knobs are read once per
process), candidates alternate over rounds so clock/power drift hits all alike.

  python tools/envab.py --cfg r8 --cands "base;TSM2X_RPT=4;TSM2X_RPT=8" --rounds 3 [--out f.json]
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CFGS = {
    "r8": (30720, 30720, 8, "double", False),
    "r16": (30720, 30720, 16, "double", False),
    "r4": (30720, 30720, 4, "double", False),
    "r2": (30720, 30720, 2, "double", False),
    "l16": (1 << 24, 16, 16, "double", True),
    "f16": (32768, 32768, 16, "single", False),
    "f8": (32768, 32768, 8, "single", False),
    "l16f": (1 << 24, 16, 16, "single", True),
    "l4": (1 << 25, 16, 4, "double", True),
    "r3": (30720, 30720, 3, "double", False),
}


def child(cfg, reps):
    import pynvml
    import torch

    import paper_2002_03258_b200 as tsm
    m, k, n, prec, czero = CFGS[cfg]
    dt = torch.float64 if prec == "double" else torch.float32
    A = tsm.colmajor_empty(m, k, dt, "cuda")
    tsm.fill_uniform(A, 1)
    B = tsm.colmajor_empty(k, n, dt, "cuda")
    tsm.fill_uniform(B, 2)
    C = tsm.colmajor_empty(m, n, dt, "cuda")
    C.zero_()
    variant = "l-opt2" if czero else "v3"
    if os.environ.get("ENVAB_TUNING"):  # e.g. small_kb=1024:tail_pct=10 (paper_2002_03258_b200.tuning)
        from paper_2002_03258_b200 import tuning
        kw = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in os.environ["ENVAB_TUNING"].split(":")}
        tuning.set_tuning(tuning.Tuning(**kw))
    if os.environ.get("ENVAB_COPY"):  # reference: a plain device copy of A's bytes (read + write)
        D = torch.empty_like(A)

        def call(*_a, **_k):
            D.copy_(A)
    else:
        call = tsm.gemm
    for _ in range(30):
        call(A, B, C, variant=variant, c_is_zero=czero)
    torch.cuda.synchronize()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    samples, stop = [], threading.Event()

    reasons = set()

    def sampler():
        fid = [pynvml.NVML_FI_DEV_POWER_INSTANT]
        while not stop.is_set():
            try:
                fv = pynvml.nvmlDeviceGetFieldValues(h, fid)[0]
                pw = fv.value.uiVal / 1000.0 if fv.nvmlReturn == 0 else pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
            except Exception:
                pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pw,
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)))
            try:
                reasons.add(int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.005)
    th = threading.Thread(target=sampler)
    th.start()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for i in range(reps):
        if i == reps // 2:
            e1.record()
        call(A, B, C, variant=variant, c_is_zero=czero)
    e2.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    half = samples[len(samples) // 2:] or [(0, 0, 0)]
    mhz = sorted(s[0] for s in half)[len(half) // 2]
    pw = sorted(s[1] for s in half)[len(half) // 2]
    mem = sorted(s[2] for s in half)[len(half) // 2]
    ms = e1.elapsed_time(e2) / (reps - reps // 2)
    bits = 0
    for r in reasons:
        bits |= r
    print(json.dumps({"ms": round(ms, 4), "sm_mhz": mhz, "power_w": pw, "mem_mhz": mem, "reasons": hex(bits)}),
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="r8")
    ap.add_argument("--cands", default="base")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=1500)
    ap.add_argument("--out", default="")
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    if args.child:
        child(args.cfg, args.reps)
        return
    cands = args.cands.split(";")
    res = {c: [] for c in cands}
    for r in range(args.rounds):
        order = cands if r % 2 == 0 else cands[::-1]
        for c in order:
            env = dict(os.environ)
            if c != "base":
                for kv in c.split(","):
                    kk, vv = kv.split("=", 1)
                    env[kk] = vv
            p = subprocess.run([sys.executable, __file__, "--child", "--cfg", args.cfg, "--reps", str(args.reps)],
                               env=env, capture_output=True, text=True, timeout=600)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
            if p.returncode != 0 or not line:
                res[c].append({"error": (p.stderr or "")[-400:]})
            else:
                res[c].append(json.loads(line[-1]))
            print(args.cfg, c, res[c][-1], flush=True)
    summary = {}
    for c, v in res.items():
        ok = [x for x in v if "ms" in x]
        if ok:
            ms = sorted(x["ms"] for x in ok)
            summary[c] = {"median_ms": ms[len(ms) // 2], "min_ms": ms[0], "runs": ok}
        else:
            summary[c] = {"runs": v}
    print(json.dumps({args.cfg: {c: {k: s[k] for k in s if k != "runs"} for c, s in summary.items()}}), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({args.cfg: summary}, fh, indent=1)


if __name__ == "__main__":
    main()
