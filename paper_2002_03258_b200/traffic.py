"""Traffic model of the kernels this package launches — the B200 counterpart of the reference's
closed-form oracle ``count_expected_loads`` (reference pkg/src/tsgemm/oracle.py:72-124) and of the
per-array counter columns of its ``run`` CSV (reference cli.py:105-124).

* :func:`paper_algorithm_loads` restates the reference's closed form for the paper's algorithms
  (V0-V3, L_OPT1/2): element loads/stores per array. The ablation kernels (csrc/ablation.cuh) run
  V0/V1/V2 exactly as written, one thread per row, so their executed global loads follow it; with
  A larger than the L2 every A load is also a DRAM read, so ``eb * loads["A"]`` is the A traffic
  ncu must see (tools/traffic_check.py, profiles/traffic_r02.json).
* :func:`stream_kernel_counts` models what the production TMA stream kernel (csrc/tsm2r_tma.cuh,
  V3 / L_OPT1 / L_OPT2) moves: A in whole-column TMA boxes once per 16-column pass, B (staged
  Bt rows) as one bulk copy per stage, C read once (unless the zero-C contract) and written once
  per row-block chunk (fp64 reductions for split row blocks).

Both return rows in the reference's column vocabulary: load_instructions, store_instructions,
load_transactions (128-byte segments), bytes_requested, bytes_transferred, gld_efficiency.
"""

from __future__ import annotations

import math
from typing import Dict

from .core import Variant

ARRAY_COLS = ["load_instructions", "store_instructions", "load_transactions", "bytes_requested",
              "bytes_transferred", "gld_efficiency"]
SEGMENT = 128  # bytes per global-memory transaction in the reference's model (GpuSpec.transaction_bytes)


def paper_algorithm_loads(variant, m: int, k: int, n: int, t1: int, t2: int, t3: int, tcf: int = 1) -> Dict:
    """Element loads/stores per array of the paper's algorithm (reference oracle.py:72-124)."""
    variant = Variant.coerce(variant)
    passes = math.ceil(n / t2)
    jsteps = math.ceil(k / t1)
    total_threads = math.ceil(m / tcf) if variant.is_tsm2l else m
    blocks = math.ceil(total_threads / t1)
    rounds = math.ceil(m / total_threads)
    if variant is Variant.V0:
        loads = {"A": m * k * n, "B": m * k * n, "C": m * k * n}
        stores = {"C": m * k * n}
    elif variant is Variant.V1:
        loads = {"A": m * k * passes, "B": m * k * n, "C": m * n}
        stores = {"C": m * n}
    elif variant in (Variant.V2, Variant.V3):
        loads = {"A": m * k * passes, "B": blocks * k * n, "C": m * n}
        stores = {"C": m * n}
    elif variant is Variant.L_OPT1:
        loads = {"A": m * k * passes, "B": blocks * rounds * k * n, "C": m * n}
        stores = {"C": m * n}
    else:
        loads = {"A": m * k * passes, "B": blocks * k * n, "C": m * n * jsteps * passes}
        stores = {"C": m * n * jsteps}
    return {"loads": loads, "stores": stores}


def _row(loads, stores, requested, transferred, transactions):
    eff = (requested / transferred) if transferred else None
    return [loads, stores, transactions, requested, transferred, eff]


def ablation_counts(variant, m: int, k: int, n: int, t1: int, t2: int, t3: int, eb: int,
                    c_is_zero: bool = True) -> Dict[str, list]:
    """Per-array counter row of the ablation kernels (V0/V1/V2, one thread per row): every warp
    access to A and C covers 32 consecutive rows of one column, every access to B is a warp
    broadcast of one element."""
    cnt = paper_algorithm_loads(variant, m, k, n, t1, t2, t3)
    out = {}
    for a in ("A", "B", "C"):
        ld, st = cnt["loads"].get(a, 0), cnt["stores"].get(a, 0)
        if a == "C" and c_is_zero and Variant.coerce(variant) is not Variant.V0:
            ld = 0  # the ablation kernels skip C's read under the zero-C contract
        if a == "B":
            warps = ld / 32  # one broadcast transaction per warp access
            out[a] = _row(ld, st, int(warps * eb), int(warps * SEGMENT), int(warps))
        else:
            req = ld * eb
            segs = ld * eb / SEGMENT if eb * 32 >= SEGMENT else ld / 32
            out[a] = _row(ld, st, int(req), int(segs * SEGMENT), int(segs))
    return out


def stream_kernel_counts(plan: Dict, m: int, k: int, n: int, eb: int, c_is_zero: bool) -> Dict[str, list]:
    """Per-array counter row of the TMA stream kernel for one call, from its launch plan
    (:func:`paper_2002_03258_b200.tuning.plan`): instructions are TMA / bulk copies (one per box
    or per stage) and C accesses per element; bytes are what those copies move."""
    R, KC, NT = plan["rows_per_block"], plan["cols_per_stage"], plan["cols_per_pass"]
    passes = math.ceil(n / 16)
    num_rb = math.ceil(m / R)
    stages = num_rb * math.ceil(k / KC)  # chunk boundaries are KC-aligned except the last
    boxes = 1 if (eb == 8 and NT in (8, 16)) or plan["consumer"] == "tc" else max(1, R // 256)
    # A: every column of every row block once per pass; TMA fetches whole 128-B segments of the
    # contiguous column runs (rows past m are zero-filled, not fetched)
    col_bytes = m * eb
    a_req = passes * k * col_bytes
    a_segs = passes * k * math.ceil(col_bytes / SEGMENT)
    A = _row(passes * stages * boxes, 0, a_req, a_segs * SEGMENT, a_segs)
    # B: the staged Bt rows (KC x NT per stage) as one bulk copy per stage, plus prep's read of B
    b_req = passes * stages * KC * NT * eb + k * n * eb
    B = _row(passes * stages + k * n, 0, b_req, math.ceil(b_req / SEGMENT) * SEGMENT, math.ceil(b_req / SEGMENT))
    # C: read once unless zero (first chunk), one write (or fp64 reduction) per chunk of a row block
    chunks = plan["nbig"] + plan["nsmall"]
    c_ld = 0 if c_is_zero else m * n
    c_st = m * n * max(1, chunks)
    c_req = c_ld * eb
    C = _row(c_ld, c_st, c_req, math.ceil(c_req / SEGMENT) * SEGMENT, math.ceil(c_req / SEGMENT))
    return {"A": A, "B": B, "C": C}
