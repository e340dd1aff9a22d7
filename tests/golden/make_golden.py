"""Generates the golden parity fixtures from the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every case it records how the inputs are generated (the reference's own RNG conventions:
``np.random.default_rng(seed)`` then ``Matrix.random`` for A then B, tests/conftest.py:37-42),
SHA-256 digests of the input bytes, and the outputs of the reference's ``run_native``
(kernels.py:391-416) and ``naive_gemm`` (oracle.py:19-37) — as digests, plus the full arrays
for small cases. The cases are the reference tests that pin results at this boundary
(SURVEY.md §8c): identity / annihilator / scalar known answers, test_kernels.py oracle cases,
the 20 ragged shapes of test_ragged_shapes_match_oracle, and a seeded draw of the acceptance
criterion-1 configurations (test_acceptance.py:36-75, with a fixed seed in place of the salted
``hash()``).

Outputs: tests/golden/golden.json, tests/golden/golden.npz
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from tsgemm.core import KernelParams, Matrix, Precision, Variant  # noqa: E402
from tsgemm.kernels import run_native  # noqa: E402
from tsgemm.oracle import max_rel_error, naive_gemm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SMALL = 1 << 12  # store full output arrays up to this many elements


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


cases = []
arrays = {}


def record(name, variant, params, A, B, C0, gen, source):
    out = run_native(variant, A, B, C0, params)
    ref = naive_gemm(A, B, C0)
    m, k, n = A.rows, A.cols, B.cols
    case = {
        "name": name,
        "source": source,
        "variant": variant.value,
        "params": {"t1": params.t1, "t2": params.t2, "t3": params.t3, "tcf": params.tcf},
        "m": m, "k": k, "n": n,
        "precision": A.precision.value,
        "gen": gen,
        "sha_A": sha(A.storage), "sha_B": sha(B.storage), "sha_C0": sha(C0.storage),
        "sha_run_native": sha(out.storage),
        "sha_naive_gemm": sha(ref.storage),
        "ref_max_rel_error": max_rel_error(out, ref),
        "run_native_bitwise_naive": bool(np.array_equal(out.storage, ref.storage)),
    }
    if m * n <= SMALL:
        arrays[name + "/run_native"] = out.storage
        arrays[name + "/naive_gemm"] = ref.storage
        case["arrays"] = True
    if gen["kind"] == "explicit":
        arrays[name + "/A"] = A.storage
        arrays[name + "/B"] = B.storage
        arrays[name + "/C0"] = C0.storage
    cases.append(case)


def random_problem(m, k, n, prec, seed):
    rng = np.random.default_rng(seed)
    A = Matrix.random(m, k, prec, rng)
    B = Matrix.random(k, n, prec, rng)
    return A, B, Matrix.zeros(m, n, prec)


D, S = Precision.DOUBLE, Precision.SINGLE


def P(variant, t1=32, t2=4, t3=4, tcf=1):
    return KernelParams(t1=t1, t2=t2, t3=t3, tcf=tcf, variant=variant)


# ---- known answers --------------------------------------------------------------------------
rng = np.random.default_rng(3)
A = Matrix.identity(64, D)
B = Matrix.random(64, 2, D, rng)
record("identity_v3", Variant.V3, P(Variant.V3, t2=2), A, B, Matrix.zeros(64, 2, D),
       {"kind": "explicit"}, "test_kernels.py:36-42")
A, _, C0 = random_problem(64, 64, 4, D, 2)
record("zero_b_v0", Variant.V0, P(Variant.V0), A, Matrix.zeros(64, 4, D), C0, {"kind": "explicit"},
       "test_kernels.py:29-33")
record("scalar_fma", Variant.V3, P(Variant.V3, t2=1), Matrix.from_2d([[2.0]], D), Matrix.from_2d([[3.0]], D),
       Matrix.from_2d([[5.0]], D), {"kind": "explicit"}, "test_oracle.py:18-22")
record("single_accumulates_double", Variant.V3, P(Variant.V3, t2=1), Matrix.from_2d([[1.0, 1.0]], S),
       Matrix.from_2d([[2.0 ** 14], [2.0 ** -11]], S), Matrix.zeros(1, 1, S), {"kind": "explicit"},
       "test_oracle.py:45-52")
# nonzero C (C += A*B semantics, README.md:88-92)
rng = np.random.default_rng(5)
A = Matrix.random(300, 70, D, rng)
B = Matrix.random(70, 5, D, rng)
C0 = Matrix.random(300, 5, D, rng)
record("nonzero_c_v3", Variant.V3, P(Variant.V3, t2=5), A, B, C0, {"kind": "explicit"}, "SPEC.md:258")

# ---- test_kernels.py oracle cases -----------------------------------------------------------
for name, m, k, n, prec, seed, variant, params, src in [
    ("v3_1024x1024x16", 1024, 1024, 16, D, 12, Variant.V3, P(Variant.V3, 128, 16, 4), "test_kernels.py:102-107"),
    ("opt1_2048x16x16", 2048, 16, 16, D, 8, Variant.L_OPT1, P(Variant.L_OPT1, 128, 16, 4, 2), "test_kernels.py:150-155"),
    ("opt2_8192x8x8", 8192, 8, 8, D, 16, Variant.L_OPT2, P(Variant.L_OPT2, 128, 8, 4, 8), "test_kernels.py:222-230"),
    ("opt2_512x96x4", 512, 96, 4, D, 14, Variant.L_OPT2, P(Variant.L_OPT2, 32, 4, 4, 2), "test_kernels.py:169-179"),
    ("opt2_1024x16x8_multipass", 1024, 16, 8, D, 51, Variant.L_OPT2, P(Variant.L_OPT2, 64, 4, 4, 4), "test_kernels.py:233-241"),
    ("native_all_128x64x4", 128, 64, 4, D, 21, Variant.V3, P(Variant.V3, 32, 4, 4), "test_kernels.py:110-117"),
]:
    A, B, C0 = random_problem(m, k, n, prec, seed)
    record(name, variant, params, A, B, C0, {"kind": "ref_rng", "seed": seed}, src)

# ---- the 20 ragged shapes of test_ragged_shapes_match_oracle (test_kernels.py:244-265) -------
rng = np.random.default_rng(99)
for i in range(20):
    m = int(rng.integers(33, 700))
    k = int(rng.integers(33, 700))
    n = int(rng.choice([2, 4, 8, 16]))
    if m % 32 == 0:
        m += 1
    if k % 32 == 0:
        k += 3
    variant = rng.choice([Variant.V2, Variant.V3, Variant.L_OPT1])
    tcf = int(rng.choice([1, 2, 3])) if variant.is_tsm2l else 1
    t2 = int(rng.choice([v for v in (1, 2, 4, 8, 16) if v <= n]))
    params = P(variant, t1=64, t2=t2, t3=int(rng.choice([1, 2, 4])), tcf=tcf)
    seed = int(rng.integers(1 << 30))
    A, B, C0 = random_problem(m, k, n, D, seed)
    record(f"ragged_{i:02d}", variant, params, A, B, C0, {"kind": "ref_rng", "seed": seed}, "test_kernels.py:244-265")

# ---- acceptance criterion 1 draws (test_acceptance.py:36-75), fixed child seeds --------------
rng = np.random.default_rng(2024)
for vi, variant in enumerate(Variant):
    for i in range(8):
        n = int(rng.choice([2, 4, 8, 16]))
        t1 = int(rng.choice([32, 64, 128]))
        t2 = int(rng.choice([v for v in (1, 2, 4, 8, 16) if v <= n]))
        t3 = int(rng.choice([v for v in (1, 2, 4, 8) if v <= t1]))
        if variant.is_tsm2l:
            m = int(rng.integers(256, 4097))
            k = n
            tcf = int(rng.choice([1, 2, 4, 8]))
        else:
            m = int(rng.integers(64, 4097))
            k = int(rng.integers(64, 2049))
            tcf = 1
        if i < 5:
            if m % t1 == 0:
                m += int(rng.integers(1, t1))
            if not variant.is_tsm2l and k % t1 == 0:
                k += int(rng.integers(1, t1))
        prec = D if i % 2 == 0 else S
        child = [2024, i, 1000 + vi]
        crng = np.random.default_rng(child)
        A = Matrix.random(m, k, prec, crng)
        B = Matrix.random(k, n, prec, crng)
        C0 = Matrix.zeros(m, n, prec)
        params = KernelParams(t1=t1, t2=t2, t3=t3, tcf=tcf, variant=variant)
        record(f"c1_{variant.value}_{i}", variant, params, A, B, C0, {"kind": "ref_rng_child", "seed": child},
               "test_acceptance.py:52-75")

with open(os.path.join(HERE, "golden.json"), "w") as fh:
    json.dump({"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg/src/tsgemm",
               "numpy": np.__version__, "cases": cases}, fh, indent=1)
np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
print(f"{len(cases)} cases, {len(arrays)} arrays")
