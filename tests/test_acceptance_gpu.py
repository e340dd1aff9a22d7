"""The reference's acceptance criterion 1 (pkg/tests/test_acceptance.py:36-75), replayed on the
B200 path: six variants x 50 seeded configurations (m up to 4096, k up to 2048, n in
{2, 4, 8, 16}, both precisions alternating, >= 20 ragged shapes per variant) through the drop-in
``run_native``, each within the reference's own bound max_rel_error <= 8*k*eps against
``naive_gemm`` (the oracle restatement, pinned to the reference by test_oracle_golden.py) — and
within the north_star's relative-Frobenius tolerance.

The reference seeds each draw with the salted ``hash(variant.value)``; a fixed
CRC32 salt stands in so the test is reproducible.
"""

import zlib

import numpy as np
import pytest

from conftest import TOL_FROB
from oracle import max_rel_error, naive_gemm, rel_frobenius

pytestmark = pytest.mark.gpu


def _draw_config(rng, variant, tsm):
    # reference test_acceptance.py:36-50
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
    return m, k, n, tsm.KernelParams(t1=t1, t2=t2, t3=t3, tcf=tcf, variant=variant)


def test_criterion_1_on_b200():
    import paper_2002_03258_b200 as tsm
    rng = np.random.default_rng(2024)
    ragged = {v: 0 for v in tsm.Variant}
    worst = 0.0
    for variant in tsm.Variant:
        salt = zlib.crc32(variant.value.encode()) % (1 << 30)
        for i in range(50):
            m, k, n, params = _draw_config(rng, variant, tsm)
            if i < 25:  # reference: force plenty of non-divisible shapes
                if m % params.t1 == 0:
                    m += int(rng.integers(1, params.t1))
                if not variant.is_tsm2l and k % params.t1 == 0:
                    k += int(rng.integers(1, params.t1))
            ragged[variant] += (m % params.t1 != 0) or (k % params.t1 != 0)
            precision = tsm.Precision.DOUBLE if i % 2 == 0 else tsm.Precision.SINGLE
            child = np.random.default_rng([2024, i, salt])
            A = tsm.Matrix.random(m, k, precision, child)
            B = tsm.Matrix.random(k, n, precision, child)
            C0 = tsm.Matrix.zeros(m, n, precision)
            out = tsm.run_native(variant, A, B, C0, params).to_2d()
            ref = naive_gemm(A.to_2d(), B.to_2d(), C0.to_2d())
            err = max_rel_error(out, ref)
            tol = 8 * k * precision.eps
            assert err <= tol, (variant, m, k, n, params, err, tol)
            assert rel_frobenius(out, ref) <= TOL_FROB[precision.value], (variant, m, k, n)
            worst = max(worst, err / tol)
        assert ragged[variant] >= 20, variant
    print(f"criterion 1 on B200: 300 configurations, worst max_rel_error / (8 k eps) = {worst:.3f}")
