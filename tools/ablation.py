"""V0 -> V1 -> V2 -> V3 ablation on B200 (the paper's Fig./PAPER.md:867).

V0/V1/V2 are the paper's algorithms compiled as written (impl="ablation", t1=128, t2=n, t3=4 —
the paper's K40c choice); V3 is the production TMA kernel. Prints one JSON line per point and
writes profiles/ablation_<tag>.json.
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402


def time_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    rows = []
    for mk in (10240, 20480):
        for n in (2, 4, 8, 16):
            A = tsm.colmajor_empty(mk, mk, torch.float64, "cuda")
            tsm.fill_uniform(A, 1)
            B = tsm.colmajor_empty(mk, n, torch.float64, "cuda")
            tsm.fill_uniform(B, 2)
            C = tsm.colmajor_empty(mk, n, torch.float64, "cuda")
            C.zero_()
            byts = 8.0 * (mk * mk + mk * n + 2 * mk * n)
            base = None
            for v in ("v0", "v1", "v2", "v3"):
                if v == "v0" and mk > 10240:
                    continue
                params = tsm.KernelParams(t1=128, t2=n, t3=4, variant=tsm.Variant.parse(v))
                impl = "ablation" if v != "v3" else "auto"
                ms = time_ms(lambda: tsm.gemm(A, B, C, variant=v, params=params, impl=impl), reps=3 if v == "v0" else 5)
                row = {"m": mk, "k": mk, "n": n, "variant": v, "ms": round(ms, 4),
                       "GBps_algorithmic": round(byts / ms / 1e6, 1), "GFLOPs": round(2.0 * mk * mk * n / ms / 1e6, 1)}
                if v == "v1":
                    base = ms
                if base:
                    row["speedup_vs_v1"] = round(base / ms, 2)
                rows.append(row)
                print(json.dumps(row), flush=True)
            del A, B, C
            torch.cuda.empty_cache()
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"ablation_{tag}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
