"""The row-sharded driver with the real sm_100a kernel: two ranks sharing cuda:0 over gloo (the
only multi-rank setup a one-GPU box allows), B broadcast from rank 0, C gathered — checked
against the whole-matrix oracle."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, k, n, out_path):
    import torch
    import torch.distributed as dist

    import paper_2002_03258_b200 as tsm
    from paper_2002_03258_b200.multi import gather_c, row_partition, run_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r0, r1 = row_partition(m, world, rank)
        A = tsm.colmajor_empty(r1 - r0, k, torch.float64, "cuda")
        tsm.fill_uniform(A, seed=1, row_offset=r0)
        C = tsm.colmajor_empty(r1 - r0, n, torch.float64, "cuda")
        tsm.fill_uniform(C, seed=3, row_offset=r0)
        B = None
        if rank == 0:
            B = tsm.colmajor_empty(k, n, torch.float64, "cuda")
            tsm.fill_uniform(B, seed=2)
        run_sharded(A, B, C, k=k, n=n)
        torch.cuda.synchronize()
        full = gather_c(C, m, n)
        if rank == 0:
            np.save(out_path, full.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,k,n", [(10000, 3000, 8), (70001, 16, 16)])
def test_sharded_gpu_matches_oracle(tmp_path, m, k, n):
    import torch.multiprocessing as mp

    from oracle import naive_gemm, rel_frobenius
    from oracle.rng import uniform_block
    out = str(tmp_path / "c.npy")
    mp.start_processes(_worker, args=(2, _free_port(), m, k, n, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    ref = naive_gemm(uniform_block(range(m), range(k), 1), uniform_block(range(k), range(n), 2),
                     uniform_block(range(m), range(n), 3))
    assert rel_frobenius(got, ref) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("nd", [1, 2, 3])
@pytest.mark.parametrize("dt_name", ["float64", "float32"])
def test_gemm_multi_device_shards(nd, dt_name):
    """tsm2x_run_multi (single process, device-resident row shards): shards on repeated devices
    (this box has one GPU) with a stream per shard; each shard bitwise equal to a one-device call
    on that shard in deterministic mode (the B copy and shard dispatch add nothing; the split of a
    row block into column chunks depends on the shard's size, so shards are not bitwise equal to
    rows of the whole-matrix call), and the assembled C within tolerance of the oracle; TSM2R with
    C += and TSM2L under the zero-C contract."""
    import numpy as np
    import torch

    import paper_2002_03258_b200 as tsm
    from oracle import naive_gemm, rel_frobenius
    dt = getattr(torch, dt_name)
    tol = 1e-12 if dt == torch.float64 else 1e-5
    for (m, k, n, czero) in [(4099, 3000, 8, False), (70001, 16, 16, True), (1000, 700, 13, False)]:
        A = tsm.colmajor_empty(m, k, dt, "cuda"); tsm.fill_uniform(A, 1)
        B = tsm.colmajor_empty(k, n, dt, "cuda"); tsm.fill_uniform(B, 2)
        C0 = tsm.colmajor_empty(m, n, dt, "cuda")
        C0.zero_() if czero else tsm.fill_uniform(C0, 3)
        variant = "l-opt2" if czero else "v3"
        A_sh, C_sh, C_one = [], [], []
        for g in range(nd):
            r0, r1 = tsm.row_range(m, nd, g)
            a = tsm.colmajor_empty(r1 - r0, k, dt, "cuda"); a.copy_(A[r0:r1])
            c = tsm.colmajor_empty(r1 - r0, n, dt, "cuda"); c.copy_(C0[r0:r1])
            c1 = tsm.colmajor_empty(r1 - r0, n, dt, "cuda"); c1.copy_(C0[r0:r1])
            tsm.gemm(a, B, c1, variant=variant, c_is_zero=czero, deterministic=True)
            A_sh.append(a); C_sh.append(c); C_one.append(c1)
        streams = [torch.cuda.Stream() for _ in range(nd)]
        torch.cuda.synchronize()
        tsm.gemm_multi(A_sh, B, C_sh, variant=variant, c_is_zero=czero, deterministic=True, streams=streams)
        torch.cuda.synchronize()
        for g in range(nd):
            assert torch.equal(C_sh[g], C_one[g]), (m, k, n, nd, g)
        got = torch.cat([c for c in C_sh], 0)
        ref = naive_gemm(A.cpu().numpy(), B.cpu().numpy(), C0.cpu().numpy())
        assert rel_frobenius(got.cpu().numpy(), ref) <= tol
    with pytest.raises(ValueError):  # a shard whose rows do not match row_range
        tsm.gemm_multi([A_sh[0][:-1]] + A_sh[1:], B, C_sh)
