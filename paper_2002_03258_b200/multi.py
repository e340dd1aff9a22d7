"""Multi-GPU driver: row-sharded TSM2R / TSM2L, one process per GPU.

A (m x k) and C (m x n) are split into contiguous row shards, rank r owning rows
[r0, r1) = row_partition(m, world, r). B (k x n, small) lives on the source rank and is
broadcast once per call over NCCL (NVLink / NVSwitch); every rank then runs the single-GPU
kernel on its shard. Rows of C are independent (reference SPEC.md:262), so there is no
reduction and no other exchange; an optional gather assembles C on one rank.

The communication is plain ``torch.distributed`` (backend "nccl" on GPUs). The local compute
is :func:`paper_2002_03258_b200.gemm`; tests inject a CPU stand-in to exercise the sharding /
broadcast / gather logic with the gloo backend on CPU.
"""

from __future__ import annotations

from typing import Callable, Optional, Tuple

ROW_ALIGN = 32  # shard boundaries on 32-row multiples keep every shard's columns 256-B aligned


def row_partition(m: int, world: int, rank: int, align: int = ROW_ALIGN) -> Tuple[int, int]:
    """Contiguous row range of ``rank``: balanced in units of ``align`` rows (the last shard
    takes the ragged tail). Every row is owned by exactly one rank."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} for world size {world}")
    blocks = (m + align - 1) // align
    b0 = blocks * rank // world
    b1 = blocks * (rank + 1) // world
    return min(m, b0 * align), min(m, b1 * align)


def colmajor_buffer(rows: int, cols: int, dtype, device):
    """A dense (rows x cols) column-major tensor (ld == rows) whose storage is one contiguous
    block, so it can be passed to collectives directly."""
    import torch
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def broadcast_b(B, k: int, n: int, dtype, device, src: int = 0, group=None, out=None):
    """Returns the k x n column-major B on every rank (rank ``src`` passes its B, others None).
    ``out`` (a dense column-major k x n buffer, e.g. from :func:`colmajor_buffer`) is reused
    instead of allocating one per call."""
    import torch.distributed as dist
    rank = dist.get_rank(group) if group is not None else dist.get_rank()
    buf = colmajor_buffer(k, n, dtype, device) if out is None else out
    if rank == src and B is not None and B.data_ptr() != buf.data_ptr():
        buf.copy_(B)
    if _host_staged(buf, group):
        host = buf.t().cpu()
        dist.broadcast(host, src=src, group=group)
        buf.t().copy_(host)
    else:
        dist.broadcast(buf.t(), src=src, group=group)  # .t() is the contiguous (n, k) storage
    return buf


def _host_staged(t, group) -> bool:
    """gloo moves CUDA tensors only for some collectives: stage through host memory there."""
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend(group) == "gloo"


def run_sharded(A_local, B, C_local, *, k: int, n: int, variant="v3", c_is_zero: bool = False, src: int = 0,
                group=None, compute: Optional[Callable] = None, b_out=None):
    """One distributed call: broadcast B from ``src``, then C_local (+)= A_local @ B on each rank.

    ``A_local``/``C_local`` are this rank's row shards (column-major). Returns (C_local, B_local).
    """
    Bl = broadcast_b(B, k, n, A_local.dtype, A_local.device, src=src, group=group, out=b_out)
    if compute is None:
        from .kernels import gemm
        gemm(A_local, Bl, C_local, variant=variant, c_is_zero=c_is_zero)
    else:
        compute(A_local, Bl, C_local, c_is_zero)
    return C_local, Bl


class RowShards:
    """The row shard a rank owns in one of the two scaling modes of the multi-GPU driver.

    * ``strong``: a fixed ``m_total`` x k problem (BASELINE configs[4]: 65536^2, n=8) split by
      :func:`row_partition` — 32-row-aligned, balanced, the last shard ragged.
    * ``weak``: every rank owns ``rows_per_rank`` rows, rank r starting at r * rows_per_rank
      (per-GPU work fixed as the world grows).

    Rows of C are independent (reference SPEC.md:262), so a shard's result is bit-identical to
    the same rows of the whole-matrix result; the only exchange is B's broadcast.
    """

    def __init__(self, scaling: str, world: int, rank: int, *, m_total: int = 0, rows_per_rank: int = 0):
        if scaling == "strong":
            if m_total < 1:
                raise ValueError("strong scaling needs m_total >= 1")
            self.r0, self.r1 = row_partition(m_total, world, rank)
            self.m_total = m_total
        elif scaling == "weak":
            if rows_per_rank < 1:
                raise ValueError("weak scaling needs rows_per_rank >= 1")
            self.r0, self.r1 = rank * rows_per_rank, (rank + 1) * rows_per_rank
            self.m_total = rows_per_rank * world
        else:
            raise ValueError(f"unknown scaling {scaling!r}")
        self.scaling, self.world, self.rank = scaling, world, rank

    @property
    def rows(self) -> int:
        return self.r1 - self.r0


def gather_c(C_local, m: int, n: int, dst: int = 0, group=None):
    """Assembles the full m x n C (column-major) on ``dst``; other ranks get None."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if group is not None else dist.get_world_size()
    rank = dist.get_rank(group) if group is not None else dist.get_rank()
    shard_rows = [row_partition(m, world, r) for r in range(world)]
    maxr = max(r1 - r0 for r0, r1 in shard_rows)
    staged = _host_staged(C_local, group)
    dev = "cpu" if staged else C_local.device
    pad = torch.zeros((n, maxr), dtype=C_local.dtype, device=dev)
    r0, r1 = shard_rows[rank]
    pad[:, : r1 - r0] = C_local.t()
    gathered = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, gather_list=gathered, dst=dst, group=group)
    if rank != dst:
        return None
    full = colmajor_buffer(m, n, C_local.dtype, C_local.device)
    for r, (a, b) in enumerate(shard_rows):
        full[a:b] = gathered[r][:, : b - a].t()
    return full
