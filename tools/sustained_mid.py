"""Sustained (back-to-back, power-capped) A/B of the mid-size work split against the previous
queue granularity, alternating blocks. Usage: python tools/sustained_mid.py"""

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
    for mk, n in ((6144, 16), (8192, 8), (8192, 16), (12288, 16)):
        A = tsm.colmajor_empty(mk, mk, torch.float64, "cuda")
        tsm.fill_uniform(A, 1)
        B = tsm.colmajor_empty(mk, n, torch.float64, "cuda")
        tsm.fill_uniform(B, 2)
        C = tsm.colmajor_empty(mk, n, torch.float64, "cuda")
        C.zero_()
        per_cta_kb = mk * mk * 8 / 148 / 1024
        old = tuning.Tuning(small_kb=max(64, min(1024, int(per_cta_kb / 48))), big_kb=min(8192, int(per_cta_kb / 6)), tail_pct=10)
        cands = {"new": tuning.Tuning(), "old": old}
        res = {k: [] for k in cands}
        for r in range(8):
            for k in (list(cands) if r % 2 == 0 else list(cands)[::-1]):
                tuning.set_tuning(cands[k])
                res[k].append(block(A, B, C, 300))
        tuning.set_tuning(None)
        print(json.dumps({"m=k": mk, "n": n, **{k: round(sorted(v)[len(v) // 2], 2) for k, v in res.items()}}), flush=True)
        del A, B, C


if __name__ == "__main__":
    main()
