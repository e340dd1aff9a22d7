"""On-device parameter sweeps (paper_2002_03258_b200.tuning) for the BASELINE shapes; writes
profiles/tuning_<tag>.json. Run under gpurun."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2002_03258_b200 import tuning  # noqa: E402


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    out = {}
    shapes = [("tsm2r_fp64_n8", 30720, 30720, 8, "double"), ("tsm2r_fp64_n16", 30720, 30720, 16, "double"),
              ("tsm2r_fp64_n2", 30720, 30720, 2, "double"), ("tsm2r_fp32_n16", 32768, 32768, 16, "single"),
              ("tsm2r_fp64_n8_4096", 4096, 4096, 8, "double")]
    for name, m, k, n, prec in shapes:
        # consumers: auto, FMA and the precision's specialised datapaths (fp64: DMMA, pipelined
        # DMMA; fp32: FFMA2, tcgen05 split tf32)
        cons = (0, 1, 2, 5) if prec == "double" else (0, 1, 3, 4)
        r = tuning.tune_tsm2r(m, k, n, prec, reps=7, consumers=cons, small_kbs=(0, 128, 1024),
                              big_kbs=(0, 1024, 8192), tail_pcts=(0, 10, 35))
        out[name] = {"best": r.best.__dict__, "best_ms": r.best_ms, "default_ms": r.default_ms,
                     "top5": sorted(r.table, key=lambda x: x["ms"])[:5], "points": len(r.table)}
        print(json.dumps({name: {k: out[name][k] for k in ("best", "best_ms", "default_ms", "points")}}), flush=True)
    r = tuning.select_tcf(1 << 24, 16, 16, "double", reps=7)
    out["tsm2l_fp64"] = {"best": r.best.__dict__, "best_ms": r.best_ms, "default_ms": r.default_ms,
                         "table": [{"tuning": t["tuning"], "ms": t["ms"]} for t in r.table]}
    print(json.dumps({"tsm2l_fp64": {k: out["tsm2l_fp64"][k] for k in ("best", "best_ms", "default_ms")}}), flush=True)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"tuning_{tag}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
