"""Kernel-only timing sweep over the BASELINE configs (dev tool; bench.py is the contract)."""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402


def time_gemm(A, B, C, impl, variant, c_is_zero, reps=10):
    s = torch.cuda.current_stream()
    for _ in range(3):
        tsm.gemm(A, B, C, impl=impl.replace("_det", ""), variant=variant, c_is_zero=c_is_zero, deterministic=impl.endswith("_det"))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for i in range(reps):
        ev[2 * i].record(s)
        tsm.gemm(A, B, C, impl=impl.replace("_det", ""), variant=variant, c_is_zero=c_is_zero, deterministic=impl.endswith("_det"))
        ev[2 * i + 1].record(s)
    torch.cuda.synchronize()
    ts = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps))
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impls", default="ldg,tma")
    ap.add_argument("--configs", default="r2,r4,r8,r16,l16,f16,r8_4096")
    ap.add_argument("--tuning", default="", help="e.g. small_kb=2048,tail_pct=10 (paper_2002_03258_b200.tuning)")
    args = ap.parse_args()
    if args.tuning:
        from paper_2002_03258_b200 import tuning
        kw = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in args.tuning.split(",")}
        tuning.set_tuning(tuning.Tuning(**kw))
    cfgs = {
        "r2": (30720, 30720, 2, torch.float64, "v3"),
        "r4": (30720, 30720, 4, torch.float64, "v3"),
        "r8": (30720, 30720, 8, torch.float64, "v3"),
        "r16": (30720, 30720, 16, torch.float64, "v3"),
        "l16": (1 << 24, 16, 16, torch.float64, "l-opt2"),
        "f16": (32768, 32768, 16, torch.float32, "v3"),
        "r8_4096": (4096, 4096, 8, torch.float64, "v3"),
    }
    for name in args.configs.split(","):
        m, k, n, dt, variant = cfgs[name]
        eb = 8 if dt == torch.float64 else 4
        A = tsm.colmajor_empty(m, k, dt, "cuda")
        tsm.fill_uniform(A, 1)
        B = tsm.colmajor_empty(k, n, dt, "cuda")
        tsm.fill_uniform(B, 2)
        C = tsm.colmajor_empty(m, n, dt, "cuda")
        C.zero_()
        czero = variant == "l-opt2"
        by = eb * (m * k + k * n + (1 if czero else 2) * m * n)
        fl = 2.0 * m * k * n
        impls = args.impls.split(",")
        for impl in impls:
            ms = time_gemm(A, B, C, impl, variant, czero)
            print(json.dumps({"cfg": name, "impl": impl, "m": m, "k": k, "n": n, "ms": round(ms, 4),
                              "GBps": round(by / ms / 1e6, 1), "GFLOPs": round(fl / ms / 1e6, 1),
                              "frac_7300": round(by / ms / 1e6 / 7300, 3)}), flush=True)
        del A, B, C
        torch.cuda.empty_cache()




def sustain_main():
    """Sustained-load probe: each config back to back for ~2 s with NVML clock/power sampling."""
    import threading
    import time

    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    cfgs = [("r8", 30720, 30720, 8, torch.float64), ("r2", 30720, 30720, 2, torch.float64),
            ("r16", 30720, 30720, 16, torch.float64), ("f16", 32768, 32768, 16, torch.float32)]
    only = os.environ.get("QB_CONFIGS")
    if only:
        cfgs = [c for c in cfgs if c[0] in only.split(",")]
    for name, m, k, n, dt in cfgs:
        A = tsm.colmajor_empty(m, k, dt, "cuda")
        tsm.fill_uniform(A, 1)
        B = tsm.colmajor_empty(k, n, dt, "cuda")
        tsm.fill_uniform(B, 2)
        C = tsm.colmajor_empty(m, n, dt, "cuda")
        C.zero_()
        for det in ((False,) if os.environ.get("QB_NO_DET") else (False, True)):
            samples = []
            stop = threading.Event()

            def sampler():
                while not stop.is_set():
                    samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
                    time.sleep(0.02)
            th = threading.Thread(target=sampler)
            th.start()
            reps = 1800
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            for i in range(reps):
                if i == reps // 2:
                    ev[1].record()
                tsm.gemm(A, B, C, deterministic=det)
            ev[2].record()
            torch.cuda.synchronize()
            stop.set()
            th.join()
            half = samples[len(samples) // 2:]
            med = sorted(s[0] for s in half)[len(half) // 2]
            pw = sorted(s[1] for s in half)[len(half) // 2]
            ms2 = ev[1].elapsed_time(ev[2]) / (reps - reps // 2)
            print(json.dumps({"sustain": name, "det": det, "ms_2nd_half": round(ms2, 4), "sm_mhz": med,
                              "power_w": pw}), flush=True)
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    if "--sustain" in sys.argv:
        sustain_main()
    else:
        main()
