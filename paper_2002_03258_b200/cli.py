"""GPU-backed experiment front-end, mirroring the reference CLI's
subcommands and CSV conventions (reference ``pkg/src/tsgemm/cli.py``: ``run`` 163-187,
``tune`` 197-214, ``model`` 234-253, ``sweep-tcf`` 265-297; atomic UTF-8/LF CSV with ``repr``
floats 67-89) — but every number here is MEASURED on the B200 (CUDA events) instead of simulated.

    python -m paper_2002_03258_b200.cli run --m 30720 --k 30720 --n 8 --variant v3 --out run.csv
    python -m paper_2002_03258_b200.cli tune --m 30720 --k 30720 --n 16 --out tune.csv
    python -m paper_2002_03258_b200.cli model --out model.csv
    python -m paper_2002_03258_b200.cli sweep-tcf --k 16 --n 16 --out sweep.csv

``run`` inputs follow the reference's convention (``default_rng([seed, shape_index])``, A then B
uniform [0,1), C0 = 0; cli.py:132-134) for shapes up to 2^26 elements of A, and the counter-based
device generator above that. The correctness column is checked against cuBLAS DGEMM on the same
device (fp64), not against the CPU oracle (the package does not depend on it).
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import tempfile
from typing import Iterable, List, Optional, Sequence

import numpy as np

from .core import KernelParams, Precision, Variant, validate_problem
from . import traffic, tuning

CATALOG_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "gpus")


def load_b200_spec() -> dict:
    """The B200 catalog entry: data/gpus/b200.yaml (the reference's GpuSpec format, readable by
    ``tsgemm.core.load_catalog``, reference core.py:390-399) merged with the B200-only measured
    figures in b200_measured.json (read vs copy bandwidth, power cap, energy per flop)."""
    import yaml
    with open(os.path.join(CATALOG_DIR, "b200.yaml"), encoding="utf-8") as fh:
        doc = yaml.safe_load(fh)
    with open(os.path.join(CATALOG_DIR, "b200_measured.json"), encoding="utf-8") as fh:
        extra = json.load(fh)
    spec = {k: v for k, v in doc.items() if k != "sources"}
    spec.update({k: v for k, v in extra.items() if k != "sources"})
    spec["core_clock_max_mhz"] = doc["core_clock"]
    return spec


B200_SPEC = load_b200_spec()


def _cell(v) -> str:
    """CSV cell text: floats as repr (round-trip exact), None as empty — the reference's CSV
    conventions (cli.py:67-72), so its readers parse these files unchanged."""
    return "" if v is None else (repr(v) if isinstance(v, float) else str(v))


def _write_csv(path: str, header: Sequence[str], rows: Iterable[Sequence]) -> None:
    """UTF-8 / LF CSV that appears complete or not at all: written to a temporary file in the
    target directory and renamed over the target."""
    target = os.path.abspath(path)
    tmp = tempfile.NamedTemporaryFile("w", encoding="utf-8", newline="", suffix=".tmp",
                                      dir=os.path.dirname(target) or ".", delete=False)
    try:
        with tmp:
            out = csv.writer(tmp, lineterminator="\n")
            out.writerow(list(header))
            out.writerows([_cell(x) for x in r] for r in rows)
        os.replace(tmp.name, target)
    except BaseException:
        try:
            os.unlink(tmp.name)
        except FileNotFoundError:
            pass
        raise


def _hbm_peak() -> float:
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(here, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return B200_SPEC["mem_bandwidth_copy_gbs"]


def _time_ms(fn, reps: int) -> float:
    import torch
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


RUN_HEADER = (["gpu", "precision", "m", "k", "n", "variant", "t1", "t2", "t3", "tcf", "shape_class", "impl",
               "consumer", "rows_per_block", "cols_per_pass", "cols_per_stage", "stages", "items", "grid",
               "time_ms", "gflops", "gbps", "hbm_frac", "check_max_rel_err", "check_rel_frobenius"]
              # the reference's per-array counter columns (cli.py:105-124), from the traffic model of
              # the kernel actually launched (traffic.py) — "counter_source" says which
              + [f"{a}_{c}" for a in ("A", "B", "C") for c in traffic.ARRAY_COLS]
              + ["counter_source", "ncu_dram_bytes_read", "ncu_dram_bytes_write", "ncu_global_ld_thread_insts",
                 "ncu_global_st_thread_insts", "ncu_kernels", "error"])
# ncu counts warp-level LDG/STG instructions; the thread-level columns are those x 32 (every lane
# of the ablation kernels' warps is active at the 32-row-multiple shapes the CLI is run on)
NCU_METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__sass_inst_executed_op_global_ld.sum",
               "smsp__sass_inst_executed_op_global_st.sum"]


def _make_inputs(prec: Precision, shape, seed: int, si: int):
    """A, B on the device by the run command's convention (see the module docstring)."""
    import torch

    from .kernels import colmajor_empty, fill_uniform
    m, k, n = shape
    dt = torch.float64 if prec is Precision.DOUBLE else torch.float32
    A = colmajor_empty(m, k, dt, "cuda")
    B = colmajor_empty(k, n, dt, "cuda")
    if m * k <= (1 << 26):
        rng = np.random.default_rng([seed, si])
        a = rng.random(m * k, dtype=np.float64).astype(prec.dtype).reshape((m, k), order="F")
        b = rng.random(k * n, dtype=np.float64).astype(prec.dtype).reshape((k, n), order="F")
        A.copy_(torch.from_numpy(a))
        B.copy_(torch.from_numpy(b))
    else:
        fill_uniform(A, seed=seed * 1000003 + si)
        fill_uniform(B, seed=seed * 1000003 + si + 7)
    return A, B


def _params_for(variant: Variant, n: int, override: dict) -> KernelParams:
    t1 = override.get("t1", 128)
    return KernelParams(t1=t1, t2=override.get("t2", n), t3=override.get("t3", min(4, t1)),
                        tcf=override.get("tcf", 1) if variant.is_tsm2l else 1, variant=variant)


def run_once(prec: Precision, shape, variant: Variant, override: dict, seed: int, si: int) -> None:
    """One call of the point, nothing else (what ncu_counters profiles)."""
    import torch

    from .kernels import colmajor_empty, gemm
    m, k, n = shape
    A, B = _make_inputs(prec, shape, seed, si)
    C = colmajor_empty(m, n, A.dtype, "cuda")
    impl = "ablation" if variant in (Variant.V0, Variant.V1, Variant.V2) else "auto"
    torch.cuda.synchronize()
    gemm(A, B, C, variant=variant, params=_params_for(variant, n, override), impl=impl, c_is_zero=True)
    torch.cuda.synchronize()


def ncu_counters(prec: Precision, shape, variant: Variant, override: dict, seed: int, si: int) -> Optional[dict]:
    """Measured counters of one call: the point re-run under Nsight Compute (``ncu`` on PATH),
    summed over the library's kernels (fill kernels excluded). None when ncu is unavailable."""
    import shutil
    import subprocess
    if shutil.which("ncu") is None:
        return None
    m, k, n = shape
    cmd = ["ncu", "--csv", "--metrics", ",".join(NCU_METRICS), "-k", "regex:^(?!fill_uniform)",
           sys.executable, "-m", "paper_2002_03258_b200.cli", "_once", "--precision", prec.value,
           "--m", str(m), "--k", str(k), "--n", str(n), "--variant", variant.value, "--seed", str(seed), "--si", str(si)]
    for f, v in override.items():
        cmd += [f"--{f}", str(v)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    rows = list(csv.reader(out.stdout.splitlines()))
    start = next((i for i, r in enumerate(rows) if r and r[0] == "ID"), None)
    if start is None:
        return None
    hdr = rows[start]
    ki, ni, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    sums, kernels = {}, set()
    for r in rows[start + 1:]:
        if len(r) <= vi or "fill_uniform" in r[ki]:
            continue
        kernels.add(r[0])
        try:
            sums[r[ni]] = sums.get(r[ni], 0.0) + float(r[vi].replace(",", ""))
        except ValueError:  # "n/a": metric not collected for this kernel
            pass
    sums["kernels"] = len(kernels)
    return sums


def _run_point(prec: Precision, shape, variant: Variant, override: dict, seed: int, si: int, reps: int,
               counters: str = "model"):
    import torch

    from .kernels import colmajor_empty, gemm
    m, k, n = shape
    base = ["B200", prec.value, m, k, n, variant.value]
    try:
        params = _params_for(variant, n, override)
        t1, t2, t3, tcf = params.t1, params.t2, params.t3, params.tcf
        params.validate_for(m, k, n)
        A, B = _make_inputs(prec, shape, seed, si)
        C = colmajor_empty(m, n, A.dtype, "cuda")
        impl = "ablation" if variant in (Variant.V0, Variant.V1, Variant.V2) else "auto"

        def call():
            C.zero_()
            gemm(A, B, C, variant=variant, params=params, impl=impl, c_is_zero=True)

        ms = _time_ms(call, reps)
        ref = (A.double() @ B.double()).cpu().numpy()
        got = C.double().cpu().numpy()
        err = float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)))
        fro = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))
        eb = prec.bytes_per_element
        byts = eb * (m * k + k * n + m * n)
        pl = tuning.plan(prec.value, m, k, n, impl=impl)
        gbps = byts / ms / 1e6
        row = base + [t1, t2, t3, tcf, validate_problem(m, k, n).value, pl["impl"], pl["consumer"],
                      pl["rows_per_block"], pl["cols_per_pass"], pl["cols_per_stage"], pl["stages"], pl["items"],
                      pl["grid"], ms, 2.0 * m * k * n / ms / 1e6, gbps, gbps / _hbm_peak(), err, fro]
        if impl == "ablation":
            cnt = traffic.ablation_counts(variant, m, k, n, t1, t2, t3, eb, c_is_zero=True)
            src = "model:paper_algorithm (oracle.py:72-124 closed form)"
        else:
            cnt = traffic.stream_kernel_counts(pl, m, k, n, eb, c_is_zero=True)
            src = "model:tma_stream_kernel"
        for a in ("A", "B", "C"):
            row += cnt[a]
        ncu = ncu_counters(prec, shape, variant, override, seed, si) if counters == "ncu" else None
        if ncu is not None:
            src += "+ncu"
            vals = [ncu.get(k_) for k_ in NCU_METRICS]
            vals[2:4] = [None if v_ is None else 32 * v_ for v_ in vals[2:4]]  # warp -> thread instructions
            row += [src] + vals + [ncu.get("kernels")]
        else:
            row += [src, None, None, None, None, None]
        row += [""]
        del A, B, C
        return row
    except Exception as exc:  # infeasible params etc.: per-row error, keep going (cli.py:155-160)
        row = base + [override.get("t1"), override.get("t2"), override.get("t3"), override.get("tcf")]
        row += [""] * (len(RUN_HEADER) - len(row) - 1)
        return row + [f"{type(exc).__name__}: {exc}"]


def cmd_run(prec: Precision, shapes, variants, override, seed, out, reps=10, counters="model") -> int:
    rows = [_run_point(prec, sh, v, override, seed, si, reps, counters) for si, sh in enumerate(shapes)
            for v in variants]
    _write_csv(out, RUN_HEADER, rows)
    return 0


TUNE_HEADER = ["gpu", "precision", "m", "k", "n", "consumer", "small_kb", "big_kb", "tail_pct", "batch_kb",
               "time_ms", "is_default", "is_best", "items", "grid", "t1", "t2", "t3"]


def cmd_tune(prec: Precision, shape, out, reps=7) -> int:
    m, k, n = shape
    r = tuning.tune_tsm2r(m, k, n, prec.value, reps=reps)
    rows = []
    for e in r.table:
        t = e["tuning"]
        pl = e["plan"]
        rows.append(["B200", prec.value, m, k, n, tuning.CONSUMERS[t["consumer"]], t["small_kb"], t["big_kb"],
                     t["tail_pct"], t["batch_kb"], e["ms"], t == tuning.Tuning().__dict__,
                     t == r.best.__dict__, pl["items"], pl["grid"], pl["t1"], pl["t2"], pl["t3"]])
    _write_csv(out, TUNE_HEADER, rows)
    return 0


MODEL_HEADER = ["gpu", "precision", "ridge_n", "mem_bandwidth_gbs", "peak_gflops", "m", "k", "n", "bytes",
                "flops", "time_mem_ms", "time_comp_ms", "bound_class", "consumer", "time_power_ms",
                "predicted_sustained_ms"]


def _consumer_for(prec: Precision, n: int) -> str:
    """The datapath the library picks for one pass of width n (tsm2x.cu pick_consumer_rt)."""
    nt = 1 if n <= 1 else 2 if n <= 2 else 4 if n <= 4 else 8 if n <= 8 else 16
    if prec is Precision.DOUBLE:
        return "dmma" if nt >= 4 else "dfma"  # 3-4 column passes run on the 8-column DMMA tile
    return "tcgen05_split_tf32" if nt == 16 else "ffma2"


def _tile_cols(prec: Precision, n: int) -> int:
    """Columns the datapath computes for a pass of width n (B zero-padded to the tile)."""
    nt = 1 if n <= 1 else 2 if n <= 2 else 4 if n <= 4 else 8 if n <= 8 else 16
    if prec is Precision.DOUBLE and nt == 4:
        return 8
    return nt


def power_bound_ms(prec: Precision, m: int, k: int, n: int) -> float:
    """Sustained time under the board power cap (DESIGN.md §4 energy model): the A stream's
    pipeline energy plus the arithmetic's, divided by the cap."""
    eb = prec.bytes_per_element
    e = B200_SPEC["pipeline_nj_per_byte"] * 1e-9 * eb * m * k + \
        B200_SPEC["energy_pj_per_flop"][_consumer_for(prec, n)] * 1e-12 * 2.0 * m * k * _tile_cols(prec, n)
    return e / B200_SPEC["power_limit_w"] * 1e3


def cmd_model(prec: Precision, out) -> int:
    """B200 roofline per n at the 30720^2 problem (the reference's model table, cli.py:234-253),
    with the corrected 2-flops-per-FMA ridge and measured peaks, plus the
    power-cap bound that sets the sustained rate on this part."""
    eb = prec.bytes_per_element
    bw = B200_SPEC["mem_bandwidth_read_gbs"] * 1e9
    pk = (B200_SPEC["peak_gflops_double"] if prec is Precision.DOUBLE else B200_SPEC["peak_gflops_single"]) * 1e9
    ridge = pk / bw * eb / 2
    rows = []
    mk = 30720
    for n in (2, 4, 8, 16, 32):
        byts = eb * (mk * mk + mk * n + 2 * mk * n)
        flops = 2.0 * mk * mk * n
        tm, tc = byts / bw, flops / pk
        tp = power_bound_ms(prec, mk, mk, n) / 1e3
        # n > 16 runs ceil(n/16) passes, each re-reading A
        passes = (n + 15) // 16
        tp = tp if passes == 1 else passes * power_bound_ms(prec, mk, mk, 16) / 1e3
        rows.append(["B200", prec.value, ridge, bw / 1e9, pk / 1e9, mk, mk, n, byts, flops, tm * 1e3, tc * 1e3,
                     "memory" if tm >= tc else "compute", _consumer_for(prec, min(n, 16)), tp * 1e3,
                     max(tm, tc, tp) * 1e3])
    _write_csv(out, MODEL_HEADER, rows)
    return 0


SWEEP_HEADER = ["gpu", "precision", "m", "k", "n", "batch_kb", "time_ms", "gbps", "is_best"]


def cmd_sweep_tcf(prec: Precision, k: int, n: int, out, ms=(10**4, 10**5, 10**6, 10**7), reps=7) -> int:
    """TSM2L dispatch-granularity sweep (the tcf analogue; reference cli.py:265-297)."""
    rows = []
    eb = prec.bytes_per_element
    for m in ms:
        r = tuning.select_tcf(m, k, n, prec.value, reps=reps)
        for e in r.table:
            t = e["tuning"]
            byts = eb * (m * k + k * n + 2 * m * n)
            rows.append(["B200", prec.value, m, k, n, t["batch_kb"], e["ms"], byts / e["ms"] / 1e6,
                         t == r.best.__dict__])
    _write_csv(out, SWEEP_HEADER, rows)
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="tsm2x", description="B200 TSM2X experiments (measured)")
    sub = p.add_subparsers(dest="command", required=True)

    def common(q):
        q.add_argument("--gpu", default="B200", help="accepted for reference compatibility; must be B200")
        q.add_argument("--precision", choices=["single", "double"], default="double")
        q.add_argument("--out", default=None)

    r = sub.add_parser("run")
    common(r)
    for d in ("m", "k", "n"):
        r.add_argument(f"--{d}", type=int, action="append", required=True)
    r.add_argument("--variant", action="append", default=None)
    for f in ("t1", "t2", "t3", "tcf"):
        r.add_argument(f"--{f}", type=int, default=None)
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--reps", type=int, default=10)
    r.add_argument("--counters", choices=["model", "ncu"], default="model",
                   help="per-array counters from the traffic model, plus Nsight Compute measurements with 'ncu'")
    o = sub.add_parser("_once")  # internal: one call of a point (profiled by ncu_counters)
    common(o)
    for d in ("m", "k", "n"):
        o.add_argument(f"--{d}", type=int, required=True)
    o.add_argument("--variant", required=True)
    for f in ("t1", "t2", "t3", "tcf"):
        o.add_argument(f"--{f}", type=int, default=None)
    o.add_argument("--seed", type=int, default=0)
    o.add_argument("--si", type=int, default=0)
    t = sub.add_parser("tune")
    common(t)
    for d in ("m", "k", "n"):
        t.add_argument(f"--{d}", type=int, required=True)
    mo = sub.add_parser("model")
    common(mo)
    s = sub.add_parser("sweep-tcf")
    common(s)
    s.add_argument("--k", type=int, default=16)
    s.add_argument("--n", type=int, default=16)
    return p


def _shapes(args) -> List[tuple]:
    L = max(len(args.m), len(args.k), len(args.n))

    def ex(xs):
        if len(xs) == 1:
            return xs * L
        if len(xs) != L:
            raise ValueError("--m/--k/--n lists must have equal length (or length 1)")
        return xs
    return list(zip(ex(args.m), ex(args.k), ex(args.n)))


def main(argv: Optional[Sequence[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    prec = Precision.parse(args.precision)
    try:
        if args.gpu.upper() != "B200":
            raise ValueError(f"this front-end measures the local B200; --gpu {args.gpu!r} is not available")
        if args.command == "run":
            override = {f: getattr(args, f) for f in ("t1", "t2", "t3", "tcf") if getattr(args, f) is not None}
            variants = [Variant.parse(v) for v in (args.variant or [])]
            return cmd_run(prec, _shapes(args), variants, override, args.seed, args.out or "run.csv", args.reps,
                           args.counters)
        if args.command == "_once":
            override = {f: getattr(args, f) for f in ("t1", "t2", "t3", "tcf") if getattr(args, f) is not None}
            run_once(prec, (args.m, args.k, args.n), Variant.parse(args.variant), override, args.seed, args.si)
            return 0
        if args.command == "tune":
            return cmd_tune(prec, (args.m, args.k, args.n), args.out or "tune.csv")
        if args.command == "model":
            return cmd_model(prec, args.out or "model.csv")
        if args.command == "sweep-tcf":
            return cmd_sweep_tcf(prec, args.k, args.n, args.out or "sweep_tcf.csv")
        raise ValueError(f"unknown command {args.command}")
    except Exception as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
