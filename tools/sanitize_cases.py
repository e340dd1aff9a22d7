"""Small calls through every kernel path (run with TSM2X_INLINE_B=0 and =1 to cover both B producers), for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck). Checks each result against a float64 torch reference so a sanitizer run is also a
parity run. Usage (GPU box):
  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402
from paper_2002_03258_b200 import tuning  # noqa: E402

CASES = [
    # (m, k, n, dtype, kwargs)
    (1000, 700, 2, torch.float64, {}),
    (1000, 700, 4, torch.float64, {}),
    (2048, 1500, 8, torch.float64, {}),               # DMMA, split row blocks
    (1500, 1300, 16, torch.float64, {}),              # DMMA, ragged rows
    (3000, 16, 16, torch.float64, {"variant": "l-opt2", "c_is_zero": True}),  # TSM2L, single-chunk
    (2048, 1500, 8, torch.float64, {"deterministic": True}),                 # ordered tickets
    (2048, 1500, 16, torch.float32, {}),              # small fp32 C +=: FFMA2, fp32 reductions into C
    (2048, 1500, 16, torch.float32, {"tc": True}),    # tcgen05 split tf32 (16 converter warps), fp64 acc + finalize
    (2048, 1500, 16, torch.float32, {"c_is_zero": True}),  # fp32 split under zero-C: fp64 acc + finalize
    (3000, 16, 16, torch.float32, {"variant": "l-opt2", "c_is_zero": True}),  # FFMA2 single-chunk, direct stores
    (3000, 16, 16, torch.float32, {"variant": "l-opt2", "c_is_zero": True, "tc": True}),  # tc32 single-chunk (deferred epilogue)
    (3000, 20, 16, torch.float32, {}),                # FFMA2 single-chunk, C += (4-column C groups)
    (2048, 1500, 8, torch.float32, {}),               # FFMA2
    (1000, 700, 40, torch.float64, {}),               # three passes (16 + 16 + 8)
    (777, 333, 8, torch.float64, {"impl": "ldg"}),    # LDG fallback
    (1001, 16, 8, torch.float64, {"impl": "tsm2l"}),  # TSM2L LDG kernel
    (512, 300, 8, torch.float64, {"impl": "ablation", "variant": "v2"}),
]


def main():
    worst = 0.0
    for m, k, n, dt, kw in CASES:
        A = tsm.colmajor_empty(m, k, dt, "cuda")
        tsm.fill_uniform(A, 1)
        B = tsm.colmajor_empty(k, n, dt, "cuda")
        tsm.fill_uniform(B, 2)
        C = tsm.colmajor_empty(m, n, dt, "cuda")
        if kw.get("c_is_zero"):
            C.zero_()
        else:
            tsm.fill_uniform(C, 3)
        ref = C.double() + A.double() @ B.double()
        kw = dict(kw)
        tc = kw.pop("tc", False)
        if tc:  # force the tensor-core consumer (auto sends single chunks to FFMA2)
            tuning.set_tuning(tuning.Tuning(consumer=4))
        tsm.gemm(A, B, C, **kw)
        if tc:
            tuning.set_tuning(None)
        torch.cuda.synchronize()
        err = ((C.double() - ref).norm() / ref.norm()).item()
        tol = 1e-12 if dt == torch.float64 else 1e-5
        print(f"{m}x{k}x{n} {str(dt)[6:]} {kw}: rel_frob {err:.2e}", flush=True)
        assert err <= tol, (m, k, n, dt, kw, err)
        worst = max(worst, err / tol)
    print(f"all {len(CASES)} cases within tolerance (worst {worst:.3f} of it)")


if __name__ == "__main__":
    main()
