import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"
# the unmodified reference installed by tools/install_reference.sh (git-ignored; travels to the GPU
# box with the snapshot, unlike /root/reference): the package and a copy of its own test modules
REFERENCE_INSTALL = os.path.join(ROOT, "baseline", "_ref")
REFERENCE_TESTS = [os.path.join(REFERENCE_INSTALL, "tsgemm_tests"), "/root/reference/pkg/tests"]


def reference_path():
    """Directory holding the importable reference ``tsgemm`` package, or None."""
    for d in (REFERENCE_INSTALL, REFERENCE_SRC):
        if os.path.isfile(os.path.join(d, "tsgemm", "__init__.py")):
            return d
    return None


def reference_tests_dir():
    for d in REFERENCE_TESTS:
        if os.path.isfile(os.path.join(d, "test_kernels.py")):
            return d
    return None


def import_reference():
    """The reference ``tsgemm`` package (importing it with its own directory on sys.path)."""
    d = reference_path()
    if d is None:
        pytest.skip("reference package not installed (tools/install_reference.sh)")
    if d not in sys.path:
        sys.path.append(d)
    import tsgemm
    return tsgemm


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built libtsm2x.so")
    config.addinivalue_line("markers", "slow: large-size GPU cases (full BASELINE configs)")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


# ---- golden fixtures ---------------------------------------------------------------------------

_golden = None


def golden():
    global _golden
    if _golden is None:
        with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
            meta = json.load(fh)
        arrays = dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))
        _golden = (meta["cases"], arrays)
    return _golden


def golden_cases():
    return golden()[0]


def regenerate(case):
    """Inputs of a golden case as 2-D F-ordered arrays (A, B, C0) using the reference's RNG
    conventions (reference tests/conftest.py:37-42, core.py:119-123)."""
    cases, arrays = golden()
    name = case["name"]
    dtype = np.float64 if case["precision"] == "double" else np.float32
    m, k, n = case["m"], case["k"], case["n"]
    gen = case["gen"]
    if gen["kind"] == "explicit":
        flat = [arrays[f"{name}/{x}"] for x in ("A", "B", "C0")]
    else:
        rng = np.random.default_rng(gen["seed"])
        a = rng.random(m * k, dtype=np.float64).astype(dtype)
        b = rng.random(k * n, dtype=np.float64).astype(dtype)
        flat = [a, b, np.zeros(m * n, dtype=dtype)]
    A = flat[0].reshape((m, k), order="F")
    B = flat[1].reshape((k, n), order="F")
    C0 = flat[2].reshape((m, n), order="F")
    return A, B, C0


def sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a).reshape(-1, order="F")).tobytes()).hexdigest()


TOL_FROB = {"double": 1e-12, "single": 1e-5}  # BASELINE.json north_star parity bar
