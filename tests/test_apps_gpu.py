"""The paper's callers on the device path: ABFT checksum encoding / checking
and k-means distances / assignment, against numpy."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _colmajor(tsm, X, torch):
    T = tsm.colmajor_empty(X.shape[0], X.shape[1], torch.float64 if X.dtype == np.float64 else torch.float32, "cuda")
    T.copy_(torch.from_numpy(X))
    return T


@pytest.mark.parametrize("m,k", [(5000, 3000), (70001, 16), (1, 1)])
def test_abft_encode_and_check(m, k):
    import torch
    import paper_2002_03258_b200 as tsm
    from paper_2002_03258_b200 import apps
    rng = np.random.default_rng(m + k)
    Ah = rng.standard_normal((m, k))
    A = _colmajor(tsm, Ah, torch)
    cs = apps.abft_encode(A).cpu().numpy()
    W = np.stack([np.ones(k), np.arange(1, k + 1)], axis=1)
    ref = Ah @ W
    assert np.allclose(cs, ref, rtol=1e-12, atol=1e-12 * np.abs(Ah).sum())
    assert apps.abft_check(A, apps.abft_encode(A)).numel() == 0
    if m > 10:
        enc = apps.abft_encode(A)
        A[7, k // 2] += 1.0  # a single corrupted element is found in its row
        assert apps.abft_check(A, enc).tolist() == [7]


@pytest.mark.parametrize("m,d,c,dt", [(100000, 16, 16, np.float64), (20000, 3000, 8, np.float64),
                                      (50000, 32, 10, np.float32)])
def test_kmeans_distances_and_assign(m, d, c, dt):
    import torch
    import paper_2002_03258_b200 as tsm
    from paper_2002_03258_b200 import apps
    rng = np.random.default_rng(d)
    Xh = rng.standard_normal((m, d)).astype(dt)
    Ch = rng.standard_normal((c, d)).astype(dt)
    X = _colmajor(tsm, Xh, torch)
    Cd = torch.from_numpy(Ch).cuda()
    D = apps.kmeans_distances(X, Cd).cpu().numpy().astype(np.float64)
    X64, C64 = Xh.astype(np.float64), Ch.astype(np.float64)
    ref = (X64 ** 2).sum(1)[:, None] - 2 * X64 @ C64.T + (C64 ** 2).sum(1)[None, :]
    tol = 1e-9 if dt == np.float64 else 2e-4
    assert np.max(np.abs(D - ref) / (np.abs(ref) + d)) <= tol
    lab = apps.kmeans_assign(X, Cd).cpu().numpy()
    ref_lab = ref.argmin(1)
    # ties within rounding aside, the assignments agree
    assert np.mean(lab == ref_lab) > 0.999
