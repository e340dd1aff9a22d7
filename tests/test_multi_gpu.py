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
