"""Sustained (back-to-back, power-capped) A/B of the mid-size work split against the previous
queue granularity, alternating blocks; "large": equal items of 1/2 or 1/3 of the per-CTA share vs
the default above the mid-size range. Usage: python tools/sustained_mid.py [large]"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402
from paper_2002_03258_b200 import tuning  # noqa: E402


def block(A, B, C, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        tsm.gemm(A, B, C)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else ""
    large = mode in ("large", "xl", "headline")
    shapes = {"large": ((12288, 8), (12288, 16), (16384, 8), (16384, 16)), "xl": ((20480, 8), (20480, 16), (24576, 8)),
              "headline": ((30720, 8), (30720, 16))}.get(
        mode, ((6144, 16), (8192, 8), (8192, 16), (12288, 16)))
    for mk, n in shapes:
        A = tsm.colmajor_empty(mk, mk, torch.float64, "cuda")
        tsm.fill_uniform(A, 1)
        B = tsm.colmajor_empty(mk, n, torch.float64, "cuda")
        tsm.fill_uniform(B, 2)
        C = tsm.colmajor_empty(mk, n, torch.float64, "cuda")
        C.zero_()
        per_cta_kb = mk * mk * 8 / 148 / 1024
        old = tuning.Tuning(small_kb=max(64, min(1024, int(per_cta_kb / 48))), big_kb=min(8192, int(per_cta_kb / 6)), tail_pct=10)
        cands = {"new": tuning.Tuning(), "old": old}
        if large:  # equal items of 1/2 and 1/3 of the per-CTA share, no tail
            cands = {"default": tuning.Tuning(), "mid16": "16", "mid64": "64",
                     "half": tuning.Tuning(small_kb=int(per_cta_kb / 2), big_kb=int(per_cta_kb / 2), tail_pct=100),
                     "third": tuning.Tuning(small_kb=int(per_cta_kb / 3), big_kb=int(per_cta_kb / 3), tail_pct=100)}
        if mode == "headline":
            cands = {"default": tuning.Tuning(), "mid64": "64"}
        res = {k: [] for k in cands}
        for r in range(8 if mode != "headline" else 12):
            for k in (list(cands) if r % 2 == 0 else list(cands)[::-1]):
                if isinstance(cands[k], str):  # the mid-size rule up to this many MB per CTA
                    os.environ["TSM2X_MID_MB"] = cands[k]
                    tuning.set_tuning(None)
                else:
                    os.environ.pop("TSM2X_MID_MB", None)
                    tuning.set_tuning(cands[k])
                res[k].append(block(A, B, C, 300))
        tuning.set_tuning(None)
        print(json.dumps({"m=k": mk, "n": n, **{k: round(sorted(v)[len(v) // 2], 2) for k, v in res.items()}}), flush=True)
        del A, B, C


if __name__ == "__main__":
    main()
