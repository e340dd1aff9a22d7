"""Item-size sweep for mid-size TSM2R problems (A within a few times L2), timed cold (L2 flushed
before every call): where per-item epilogues and the tail, not HBM, set the time.
Usage: python tools/midsize_sweep.py > gpurun_out/midsize.jsonl"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2002_03258_b200 import tuning  # noqa: E402


def main():
    shapes = [(2048, 16, "double"), (4096, 8, "double"), (4096, 16, "double"), (8192, 8, "double"),
              (8192, 16, "double"), (4096, 16, "single"), (16384, 8, "double")]
    for mk, n, prec in shapes:
        r = tuning.tune_tsm2r(mk, mk, n, prec, reps=15, consumers=(0,), small_kbs=(0, 256, 512, 1024),
                              big_kbs=(0, 512, 1024, 2048), tail_pcts=(0, 10, 35, 100))
        top = sorted(r.table, key=lambda x: x["ms"])[:6]
        print(json.dumps({"m=k": mk, "n": n, "precision": prec, "default_us": round(r.default_ms * 1e3, 1),
                          "best_us": round(r.best_ms * 1e3, 1),
                          "top": [{"t": {k: v for k, v in x["tuning"].items() if v}, "us": round(x["ms"] * 1e3, 1),
                                   "items": x["plan"]["items"], "grid": x["plan"]["grid"]} for x in top]}), flush=True)


if __name__ == "__main__":
    main()
