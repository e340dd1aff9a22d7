"""API contracts on the GPU: run-to-run reproducibility of the drop-in, layout checks, CUDA-graph
capture rules, sub-view tails, and the multi-GPU bench path through NCCL (torchrun, world 1 —
the only world a one-GPU box allows — so the NCCL branch of bench.py / multi.py executes)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from oracle import naive_gemm, rel_frobenius

pytestmark = pytest.mark.gpu


def _tsm():
    import paper_2002_03258_b200 as tsm
    return tsm


def test_run_native_is_bitwise_reproducible():
    """run_native defaults to the ordered combine (TSM2X_FLAG_DETERMINISTIC through the host path):
    repeated calls on a shape with split row blocks and several H2D column slabs return the same
    bits; deterministic=False is within tolerance of it."""
    tsm = _tsm()
    rng = np.random.default_rng(5)
    m, k, n = 2048, 20000, 8  # 4 row blocks (split across CTAs), 328 MB of A -> 2 column slabs
    A = rng.random((m, k))
    B = rng.random((k, n))
    C0 = rng.random((m, n))
    D = tsm.Precision.DOUBLE
    Am, Bm, Cm = tsm.Matrix.from_2d(A, D), tsm.Matrix.from_2d(B, D), tsm.Matrix.from_2d(C0, D)
    p = tsm.KernelParams(t1=128, t2=8, t3=4)
    outs = [tsm.run_native(tsm.Variant.V3, Am, Bm, Cm, p) for _ in range(3)]
    assert outs[0] == outs[1] == outs[2]
    fast = tsm.run_native(tsm.Variant.V3, Am, Bm, Cm, p, deterministic=False)
    assert rel_frobenius(fast.to_2d(), outs[0].to_2d()) <= 1e-14
    ref = naive_gemm(A[:256], B, C0[:256])
    assert rel_frobenius(outs[0].to_2d()[:256], ref) <= 1e-12


def test_gemm_rejects_overlapping_layouts():
    import torch
    tsm = _tsm()
    A = tsm.colmajor_empty(256, 64, torch.float64, "cuda")
    C = tsm.colmajor_empty(256, 8, torch.float64, "cuda")
    Bexp = torch.ones(64, 1, dtype=torch.float64, device="cuda").expand(64, 8)
    with pytest.raises(ValueError):
        tsm.gemm(A, Bexp, C)
    Cexp = torch.zeros(256, 1, dtype=torch.float64, device="cuda").expand(256, 8)
    B = tsm.colmajor_empty(64, 8, torch.float64, "cuda")
    with pytest.raises(ValueError):
        tsm.gemm(A, B, Cexp)


def test_capture_refuses_workspace_growth_then_replays():
    """A capture on a fresh stream (empty workspace) is refused with a clear error instead of
    baking graph-owned memory into the workspace; after one eager call the same capture works
    and replays correctly."""
    import torch
    tsm = _tsm()
    m, k, n = 4096, 4096, 8
    A = tsm.colmajor_empty(m, k, torch.float64, "cuda")
    tsm.fill_uniform(A, seed=1)
    B = tsm.colmajor_empty(k, n, torch.float64, "cuda")
    tsm.fill_uniform(B, seed=2)
    C = tsm.colmajor_empty(m, n, torch.float64, "cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(RuntimeError, match="capture"):
        with torch.cuda.graph(g, stream=s):
            tsm.gemm(A, B, C, c_is_zero=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        tsm.gemm(A, B, C, c_is_zero=True)  # eager call sizes the stream's workspace
    torch.cuda.synchronize()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        tsm.gemm(A, B, C, c_is_zero=True)
    C.fill_(float("nan"))
    g2.replay()
    torch.cuda.synchronize()
    assert rel_frobenius(C.cpu().numpy(), (A @ B).cpu().numpy()) <= 1e-12


_SUBVIEW = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2002_03258_b200 as tsm
from oracle import rel_frobenius
# exact-size allocations (no caching allocator): a sub-view ending at its buffer's end
for dt, m0, rows in ((torch.float64, 40, 64), (torch.float32, 40, 64), (torch.float64, 7, 64)):
    k, n = 3000, (8 if dt == torch.float64 else 16)
    big = torch.rand(k, rows, dtype=dt, device="cuda").t()   # rows x k column-major, ld = rows
    A = big[m0:rows]                                         # m = rows - m0, ends at the buffer end
    B = torch.rand(k, n, dtype=dt, device="cuda").t().contiguous().t()
    C = torch.zeros(n, A.shape[0], dtype=dt, device="cuda").t()
    tsm.gemm(A, B, C, c_is_zero=True)
    torch.cuda.synchronize()
    err = rel_frobenius(C.double().cpu().numpy(), (A.double() @ B.double()).cpu().numpy())
    assert err <= (1e-12 if dt == torch.float64 else 1e-5), (dt, m0, err)
print("subview ok")
"""


def test_subview_tail_stays_in_allocation():
    """A = big[40:64, :] with big an exact-size allocation (PYTORCH_NO_CUDA_MEMORY_CACHING): the
    3-D TMA layouts would read rows past m in the last column, outside the allocation; the library
    checks the allocation range and falls back to the 2-D map there."""
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    out = subprocess.run([sys.executable, "-c", _SUBVIEW, ROOT], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and "subview ok" in out.stdout, out.stderr[-3000:]


def _json_line(text):
    lines = [l for l in text.splitlines() if l.startswith("{")]
    assert len(lines) == 1, text[-3000:]
    return json.loads(lines[0])


@pytest.mark.slow
def test_bench_strong_scaling_nccl_world1():
    """BASELINE configs[4] (65536^2 fp64, n=8, strong row split) through torchrun with the NCCL
    backend: the B broadcast runs through NCCL inside every timed step."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "1", "--workload", "tsm2r_fp64_n8_65536",
           "--steps", "5", "--warmup", "3", "--e2e-steps", "0", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                         env=dict(os.environ, NCCL_DEBUG="INFO"))
    assert out.returncode == 0, out.stderr[-4000:]
    d = _json_line(out.stdout)
    assert d["scaling"] == "strong" and d["n_gpus"] == 1
    assert d["config"]["m_total"] == 65536 and d["config"]["m_per_gpu"] == 65536
    assert d["comm"]["backend"] == "nccl" and d["comm"]["bytes"] == 65536 * 8 * 8
    assert d["comm"]["ms_per_step"] >= 0 and d["value"] > 5000
    log = out.stdout + out.stderr  # torchrun workers print NCCL's log to stdout
    assert "NCCL INFO" in log and "nranks 1" in log.lower()


@pytest.mark.slow
def test_bench_config1_flushed():
    out = subprocess.run([sys.executable, "bench.py", "--workload", "tsm2r_fp64_n8_4096", "--steps", "20", "--warmup",
                          "3", "--e2e-steps", "1", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    d = _json_line(out.stdout)
    assert "flushed" in d["config"]["l2"] and d["value"] > 1000
    assert d["e2e"]["drop_in"]["value"] > 0


def test_release_cached_memory_frees_stream_workspaces():
    """Workspaces are per (device, stream) and kept across calls; release_cached_memory frees them
    (a process creating many streams otherwise keeps every stream's workspace)."""
    import torch
    tsm = _tsm()
    m, k, n = 65536, 4096, 16  # fp32 split row blocks: Bt + an fp64 accumulator per stream
    A = tsm.colmajor_empty(m, k, torch.float32, "cuda")
    tsm.fill_uniform(A, seed=1)
    B = tsm.colmajor_empty(k, n, torch.float32, "cuda")
    tsm.fill_uniform(B, seed=2)
    C = tsm.colmajor_empty(m, n, torch.float32, "cuda")
    tsm.release_cached_memory()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    streams = [torch.cuda.Stream() for _ in range(12)]
    for s in streams:
        with torch.cuda.stream(s):
            tsm.gemm(A, B, C, c_is_zero=True)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 >= 12 * (m * n * 8)  # every stream kept at least its accumulator
    tsm.release_cached_memory()
    free2 = torch.cuda.mem_get_info()[0]
    assert free2 >= free0 - (64 << 20)
    tsm.gemm(A, B, C, c_is_zero=True)  # the library re-allocates on demand
    torch.cuda.synchronize()
    ref = (A.double() @ B.double())
    assert rel_frobenius(C.double().cpu().numpy(), ref.cpu().numpy()) <= 1e-5


def test_overlapping_c_rejected():
    """C is written while A and B are read: a C that overlaps A or B is a ValueError, with no
    device work (a disjoint sub-view of the same buffer is fine)."""
    import torch
    import paper_2002_03258_b200 as tsm
    buf = tsm.colmajor_empty(4096, 64, torch.float64, "cuda")
    tsm.fill_uniform(buf, 1)
    A = buf[:, 0:32]
    B = tsm.colmajor_empty(32, 8, torch.float64, "cuda")
    tsm.fill_uniform(B, 2)
    with pytest.raises(ValueError, match="overlaps"):
        tsm.gemm(A, B, buf[:, 24:32])  # C = the last 8 columns of A
    with pytest.raises(ValueError, match="overlaps"):
        tsm.gemm(buf[:32, 32:64], B, buf[:32, 40:48])
    C = buf[:, 40:48]  # columns 40-47: disjoint from A (0-31)
    ref = C.clone() + A @ B
    tsm.gemm(A, B, C)
    torch.cuda.synchronize()
    assert torch.allclose(C, ref, rtol=1e-12, atol=0)
