"""Multi-process (world_size 2, gloo, CPU) coverage of the row-sharded driver: partition,
B broadcast, local compute on each shard, gather — checked bitwise against the whole-matrix
oracle (rows are independent, so sharding must not change a single bit)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2002_03258_b200.multi import RowShards, colmajor_buffer, gather_c, row_partition, run_sharded


def test_row_partition_covers_exactly():
    for m in (1, 31, 32, 33, 1000, 30720, 65536, 123457):
        for world in (1, 2, 3, 4, 8):
            spans = [row_partition(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1
            for a0, _ in spans:
                assert a0 % 32 == 0
    with pytest.raises(ValueError):
        row_partition(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_compute(A, B, C, c_is_zero):
    from oracle import naive_gemm
    C0 = np.zeros(tuple(C.shape)) if c_is_zero else C.numpy()
    C.copy_(torch.from_numpy(naive_gemm(A.numpy(), B.numpy(), C0.astype(A.numpy().dtype))))


def _worker(rank, world, port, m, k, n, c_is_zero, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.rng import uniform_block
        r0, r1 = row_partition(m, world, rank)
        A = torch.from_numpy(uniform_block(range(r0, r1), range(k), 1)).t().contiguous().t()
        C = torch.from_numpy(uniform_block(range(r0, r1), range(n), 3)).t().contiguous().t()
        B = torch.from_numpy(uniform_block(range(k), range(n), 2)) if rank == 0 else None
        C, Bl = run_sharded(A, B, C, k=k, n=n, c_is_zero=c_is_zero, compute=_oracle_compute)
        assert np.array_equal(Bl.numpy(), uniform_block(range(k), range(n), 2))
        full = gather_c(C, m, n)
        if rank == 0:
            np.save(out_path, full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,k,n,c_is_zero", [(1000, 77, 8, False), (4099, 16, 16, True)])
def test_sharded_equals_whole(tmp_path, m, k, n, c_is_zero):
    from oracle import naive_gemm
    from oracle.rng import uniform_block
    out = str(tmp_path / "c.npy")
    mp.start_processes(_worker, args=(2, _free_port(), m, k, n, c_is_zero, out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    C0 = np.zeros((m, n)) if c_is_zero else uniform_block(range(m), range(n), 3)
    whole = naive_gemm(uniform_block(range(m), range(k), 1), uniform_block(range(k), range(n), 2), C0)
    assert np.array_equal(got, whole)


def test_row_shards_modes():
    for world in (1, 2, 3, 8):
        strong = [RowShards("strong", world, r, m_total=65536) for r in range(world)]
        assert sum(s.rows for s in strong) == 65536 and strong[0].r0 == 0 and strong[-1].r1 == 65536
        weak = [RowShards("weak", world, r, rows_per_rank=30720) for r in range(world)]
        assert all(s.rows == 30720 and s.m_total == 30720 * world for s in weak)
    with pytest.raises(ValueError):
        RowShards("diagonal", 2, 0, m_total=10)


def _strong_worker(rank, world, port, m, k, n, steps, out_path):
    """bench.py's strong-scaling step on CPU: RowShards split, B broadcast into a reused buffer
    every step, local compute, gather."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.rng import uniform_block
        sh = RowShards("strong", world, rank, m_total=m)
        A = torch.from_numpy(uniform_block(range(sh.r0, sh.r1), range(k), 1)).t().contiguous().t()
        C = torch.from_numpy(uniform_block(range(sh.r0, sh.r1), range(n), 3)).t().contiguous().t()
        B = torch.from_numpy(uniform_block(range(k), range(n), 2)).t().contiguous().t() if rank == 0 else None
        bbuf = colmajor_buffer(k, n, torch.float64, "cpu")
        for _ in range(steps):  # C accumulates steps x A*B (C += A*B each step)
            C, Bl = run_sharded(A, B, C, k=k, n=n, compute=_oracle_compute, b_out=bbuf)
            assert Bl.data_ptr() == bbuf.data_ptr()
        full = gather_c(C, m, n)
        if rank == 0:
            np.save(out_path, full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 1000), (3, 1000), (3, 4133)])
def test_strong_split_equals_whole(tmp_path, world, m):
    """Uneven strong splits (ragged last shard, world 2 and 3) are bitwise the whole-matrix rows."""
    from oracle import naive_gemm
    from oracle.rng import uniform_block
    k, n, steps = 96, 8, 2
    out = str(tmp_path / "c.npy")
    mp.start_processes(_strong_worker, args=(world, _free_port(), m, k, n, steps, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    A, B = uniform_block(range(m), range(k), 1), uniform_block(range(k), range(n), 2)
    whole = uniform_block(range(m), range(n), 3)
    for _ in range(steps):
        whole = naive_gemm(A, B, whole)
    assert np.array_equal(got, whole)


def test_c_row_range_matches_row_partition():
    """tsm2x_row_range (the C ABI's shard split for tsm2x_run_multi / tsm2x_run_host_multi) is
    multi.row_partition, for ragged and tiny m."""
    from paper_2002_03258_b200 import row_range
    from paper_2002_03258_b200.multi import row_partition
    for m in (0, 1, 31, 32, 33, 1000, 4099, 65536, 70001):
        for nd in (1, 2, 3, 5, 8):
            got = [row_range(m, nd, g) for g in range(nd)]
            assert got == [row_partition(m, nd, g) for g in range(nd)], (m, nd)
            assert got[0][0] == 0 and got[-1][1] == m
    assert row_range(100, 2, 5) == (0, 0)  # out-of-range shard: empty
