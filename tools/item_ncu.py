"""Work-item candidates for mid-size TSM2R shapes, timed by ncu (cold caches, ns resolution; CUDA
event timing on these ~20-100 us calls is quantised to ~2 us). Run under ncu:
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tsm2r_stream --csv \
      python tools/item_ncu.py > gpurun_out/item_ncu.csv
then: python tools/item_ncu.py --report gpurun_out/item_ncu.csv"""

import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

REPS = 3


def candidates():
    from paper_2002_03258_b200.tuning import Tuning
    out = []
    for mk, n, prec in ((2048, 16, "double"), (4096, 8, "double"), (4096, 16, "double"), (6144, 8, "double"),
                        (6144, 16, "double"), (8192, 8, "double"), (8192, 16, "double"), (6144, 16, "single"), (12288, 8, "double"), (12288, 16, "double"),
                        (16384, 16, "double")):
        eb = 8 if prec == "double" else 4
        per_cta_kb = mk * mk * eb / 148 / 1024
        cands = [Tuning()]
        for f in (0.5, 1.0, 1.1, 1.3, 2.0):
            kb = int(per_cta_kb * f)
            cands.append(Tuning(small_kb=kb, big_kb=kb, tail_pct=100))
        cands += [Tuning(small_kb=512, big_kb=1024, tail_pct=35), Tuning(small_kb=256)]
        out += [((mk, n, prec), t) for t in cands]
    return out


def run():
    import torch

    import paper_2002_03258_b200 as tsm
    from paper_2002_03258_b200 import tuning
    cur = None
    for (mk, n, prec), t in candidates():
        if cur != (mk, n, prec):
            dt = torch.float64 if prec == "double" else torch.float32
            A = tsm.colmajor_empty(mk, mk, dt, "cuda")
            tsm.fill_uniform(A, 1)
            B = tsm.colmajor_empty(mk, n, dt, "cuda")
            tsm.fill_uniform(B, 2)
            C = tsm.colmajor_empty(mk, n, dt, "cuda")
            C.zero_()
            cur = (mk, n, prec)
        tuning.set_tuning(t)
        for _ in range(REPS):
            tsm.gemm(A, B, C)
        torch.cuda.synchronize()
    tuning.set_tuning(None)


def report(path):
    from paper_2002_03258_b200 import tuning
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
    durs = [float(r[-1].replace(",", "")) for r in rows]
    unit = rows[0][-2] if rows else "ns"
    scale = 1e-3 if unit == "ns" else 1.0
    res = {}
    for i, (shape, t) in enumerate(candidates()):
        d = sorted(durs[i * REPS:(i + 1) * REPS])
        if len(d) < REPS:
            break
        tuning.set_tuning(t)
        p = tuning.plan(shape[2], shape[0], shape[0], shape[1])
        res.setdefault(str(shape), []).append({"t": {k: v for k, v in t.__dict__.items() if v}, "us": round(d[1] * scale, 2),
                                               "items": p["items"], "grid": p["grid"]})
    tuning.set_tuning(None)
    for s, v in res.items():
        print(json.dumps({"shape": s, "default_us": v[0]["us"], "cands": sorted(v, key=lambda x: x["us"])}))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--report":
        report(sys.argv[2])
    else:
        run()
