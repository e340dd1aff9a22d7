#!/usr/bin/env python
"""Benchmark — BASELINE.json metric "TSM2R/TSM2L fp64 GFLOP/s and achieved HBM GB/s (% roofline)".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ...]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (N=1): BASELINE configs[1] at its headline point — TSM2R fp64, reference naming
A m x k = 30720 x 30720, B k x n = 30720 x 8 (BASELINE naming n=30720, k=8), C m x n,
C += A*B. One "step" = one full TSM2R call over that problem with A resident in HBM
(7.55 GB, 60x the 126 MB L2, so no L2 flush is needed between steps).
N > 1 (torchrun): the default workload scales weakly — every rank owns a 30720-row shard of a
(30720*N) x 30720 A. --workload tsm2r_fp64_n8_65536 is BASELINE configs[4] as specified: one
65536 x 65536 A, rows split over the ranks by multi.row_partition (strong scaling). Either way
each rank generates its shard on its device with the shared counter-based generator, B is
broadcast from rank 0 over NCCL inside every step (the path's one exchange; timed separately
as "comm"), then each rank runs the kernel on its shard; no reduction (rows are independent,
reference SPEC.md:262). Under torchrun the process group exists at N=1 too, so the NCCL path
runs at every N. Time = max over ranks of the device-event time of the K steps.
Workloads whose A is under 4x the L2 (tsm2r_fp64_n8_4096) flush the L2 between steps and time
each step with its own events.

The JSON line also carries: roofline (dominant kernel; CUDA events bracketing each call's launches
— prep_dyn when the call has one, the stream kernel, tsm2_finalize for fp32 split passes — so
kernel_ms is the call's device time, a conservative denominator),
cpu_baseline (the reference CPU path restated in numpy — oracle/ — on a bounded row sample, rank 0,
N=1), e2e (same metric through the host-buffer C ABI tsm2x_run_host with pinned host buffers,
H2D of A and D2H of C inside the timed region; at N=1 also e2e.drop_in: the reference user's call
run_native(Variant, Matrix, ...) on pageable numpy storage), comm (the B broadcast), clocks (NVML samples during the timed region),
gpu_launches (libtsm2x launches in the timed region).

--impl reference: the reference's CPU implementation of the path (run_native's vectorised body,
kernels.py:391-416, restated in oracle/reference.py — the reference is pure Python and has no
compiled form) on all host threads, rank 0 only, bounded row sample per step.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TSM2R/TSM2L fp64 GFLOP/s and achieved HBM GB/s (% roofline) at 1/2/4/8 B200"
UNIT = "GFLOP/s"

WORKLOADS = {
    # name: (rows m — per GPU for weak scaling, whole problem for strong — k, n, precision,
    #        variant, c_is_zero, description, scaling)
    "tsm2r_fp64_n8": (30720, 30720, 8, "double", "v3", False,
                      "TSM2R fp64, ref (m,k,n)=(30720,30720,8) = BASELINE configs[1] n=30720,k=8; C += A*B", "weak"),
    "tsm2r_fp64_n2": (30720, 30720, 2, "double", "v3", False, "TSM2R fp64 BASELINE configs[1] k=2", "weak"),
    "tsm2r_fp64_n4": (30720, 30720, 4, "double", "v3", False, "TSM2R fp64 BASELINE configs[1] k=4", "weak"),
    "tsm2r_fp64_n16": (30720, 30720, 16, "double", "v3", False, "TSM2R fp64 BASELINE configs[1] k=16", "weak"),
    "tsm2l_fp64": (1 << 24, 16, 16, "double", "l-opt2", True,
                   "TSM2L fp64 A 2^24x16, B 16x16, C = A*B (L_OPT2 zero-C contract), BASELINE configs[2]", "weak"),
    "tsm2r_fp32_n16": (32768, 32768, 16, "single", "v3", False, "TSM2R fp32 BASELINE configs[3]", "weak"),
    "tsm2r_fp64_n8_65536": (65536, 65536, 8, "double", "v3", False,
                            "TSM2R fp64 ref (m,k,n)=(65536,65536,8) = BASELINE configs[4], rows of A sharded over "
                            "the GPUs (strong scaling), B broadcast over NCCL every step", "strong"),
    "tsm2r_fp64_n8_4096": (4096, 4096, 8, "double", "v3", False,
                           "TSM2R fp64 ref (m,k,n)=(4096,4096,8) = BASELINE configs[0] (the oracle config); L2 "
                           "flushed between steps", "weak"),
}
L2_BYTES = 126 * (1 << 20)


def spec(wl):
    """(m, k, n, prec, variant, c_is_zero, desc, scaling) of a workload."""
    return WORKLOADS[wl]


def flush_l2_needed(m, k, eb):
    """Inputs smaller than 4x the L2 get an L2 flush between timed steps (timing rules)."""
    return m * k * eb < 4 * L2_BYTES


def bench_config(wl, world):
    """The `config` object — identical in both arms and on every N, so the driver can match them."""
    from paper_2002_03258_b200.multi import RowShards
    m, k, n, prec, variant, c_is_zero, desc, scaling = spec(wl)
    eb = 8 if prec == "double" else 4
    sh = RowShards(scaling, world, 0, m_total=m, rows_per_rank=m)
    a_gb = sh.rows * k * eb / 1e9
    return {"workload": desc, "scaling": scaling, "m_total": sh.m_total, "m_per_gpu": sh.rows, "k": k, "n": n,
            "precision": prec, "variant": variant,
            "naming": "reference (m,k,n), skinny n (SURVEY.md G1)",
            "parallelism": f"row-shard x{world}" + (", B broadcast per step (NCCL)" if world > 1 else ""),
            "l2": (f"L2 flushed between steps by reading 252 MB, outside the per-step events (A {a_gb:.3f} GB per GPU "
                   "< 4 x 0.126 GB L2)" if flush_l2_needed(sh.rows, k, eb)
                   else f"inputs larger than L2 (A {a_gb:.2f} GB per GPU vs 0.126 GB L2), no flush"),
            "bytes_form": "eb*(mk+kn+mn) C write-only" if c_is_zero else "eb*(mk+kn+2mn) C read+write"}


def algorithmic(m, k, n, eb, c_is_zero):
    """flops = 2mkn; bytes = eb*(mk + kn + 2mn) (C read+write) or eb*(mk+kn+mn)."""
    flops = 2.0 * m * k * n
    byts = eb * (m * k + k * n + (1 if c_is_zero else 2) * m * n)
    return flops, byts


def kernel_name(prec, m, k, n, c_is_zero):
    """The dominant kernel this workload launches, from the library's own plan (tsm2x_plan_for)."""
    from paper_2002_03258_b200 import tuning
    p = tuning.plan(prec, m, k, n)
    if p["consumer"] == "tc":
        return ("tsm2r_stream_tc32 (tcgen05 kind::tf32, split precision A.[B|lo B] + lo(A).B, accumulators in TMEM; "
                "dynamic items)")
    names = {"dmma": "DMMA m8n8k4", "dmmap": "DMMA m8n8k4, k-step software pipeline", "fma": "DFMA/FFMA",
             "ffma2": "packed FFMA2"}
    # bench's operands come from colmajor_empty (lda padded to 32): the DMMA passes read A through
    # the swizzled 3-D TMA layout unless TSM2X_SWZ=0
    swz = p["consumer"] in ("dmma", "dmmap") and os.environ.get("TSM2X_SWZ", "1") != "0"
    return f"tsm2r_stream_tma ({names.get(p['consumer'], p['consumer'])} consumer" + \
        ("; swizzled A (3-D TMA box, 128B swizzle)" if swz else "") + "; dynamic items" + \
        ("; single-chunk row blocks)" if p["nbig"] == 0 and p["nsmall"] == 1 else ")")


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(workload):
    """dram bytes read+write per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        e = d.get(workload)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clocks"}

    def __init__(self, device_index, period=0.01):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        busy = [s for s in self.samples] or [0]
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------
def cpu_sample_inputs(m, k, n, prec, c_is_zero, rows, cols):
    """A (rows x cols) corner of the workload's A (+ matching B rows, C rows), regenerated on the
    host by the shared generator. The reference's per-element work (and so its GFLOP/s) is the
    same for any such sample; sampling columns keeps each numpy call as large as in the full run."""
    import numpy as np

    from oracle.rng import uniform_block
    dt = np.float64 if prec == "double" else np.float32
    rows, cols = min(rows, m), min(cols, k)
    A = uniform_block(range(rows), range(cols), 1, dt)
    B = uniform_block(range(cols), range(n), 2, dt)
    C = np.zeros((rows, n), dt) if c_is_zero else uniform_block(range(rows), range(n), 3, dt)
    return A, B, C


def cpu_time(A, B, C, threads, cols=None):
    """Seconds for the reference CPU path (oracle restatement of run_native) on the first cols."""
    from oracle import run_native_port_threaded
    cols = A.shape[1] if cols is None else cols
    t0 = time.perf_counter()
    run_native_port_threaded(A[:, :cols], B[:cols], C, threads=threads)
    return time.perf_counter() - t0


def cpu_sample_shape(m, k, max_elems=1 << 25):
    """Rows x cols of the CPU sample: whole rows up to 30720 (TSM2R) and as many columns as fit
    max_elems; for TSM2L (tiny k) all columns and a row slab."""
    if k > 64:
        rows = min(m, 30720)
        cols = min(k, max(1, max_elems // rows))
    else:
        cols = k
        rows = min(m, max(1, max_elems // k))
    return rows, cols


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference_arm(args, wl):
    m, k, n, prec, variant, c_is_zero, desc, scaling = spec(wl)
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = host_threads()
    rows, cols = cpu_sample_shape(m, k)
    A, B, C = cpu_sample_inputs(m, k, n, prec, c_is_zero, rows, cols)
    # calibrate the columns per step so warmup + steps finish in about two minutes
    c0 = min(cols, 64)
    t0 = min(cpu_time(A, B, C, threads, c0) for _ in range(2))
    per_step_budget = max(0.05, 120.0 / max(1, args.steps + args.warmup))
    cs = int(max(min(cols, 8), min(cols, c0 * per_step_budget / max(t0, 1e-6))))
    for _ in range(args.warmup):
        cpu_time(A, B, C, threads, cs)
    times = [cpu_time(A, B, C, threads, cs) for _ in range(args.steps)]
    tot = sum(times)
    value = 2.0 * rows * cs * n * len(times) / tot / 1e9
    sample = (f"A[:{rows}, :{cs}] of the {m} x {k} A per step (n={n}, {prec}); reference run_native body "
              f"(kernels.py:391-416) restated in numpy (oracle/reference.py), row slabs on {threads} threads "
              f"(the reference itself is single-threaded numpy, so this arm is {threads}x generous to it); the "
              f"rate is per element of A, linear in the columns sampled, so it extrapolates to the full k")
    pkg = reference_package_rate(m, k, n, prec, c_is_zero)
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(times), 3),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f64" if prec == "double" else "f32", "data": "synthetic (counter-based U[0,1))",
            "config": bench_config(wl, args.gpus), "sample": sample,
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_package": pkg}
    print(json.dumps(line), flush=True)


def reference_package_rate(m, k, n, prec, c_is_zero, budget_s=8.0):
    """The UNMODIFIED reference (baseline/_ref, tools/install_reference.sh): tsgemm.kernels.run_native
    on a bounded sample of the workload, single-threaded as it is written — beside the port's
    all-threads rate, to show the port is the reference's speed per core, not slower."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isfile(os.path.join(ref_dir, "tsgemm", "__init__.py")):
        return None
    import numpy as np
    if ref_dir not in sys.path:
        sys.path.append(ref_dir)
    from tsgemm.core import KernelParams, Matrix, Precision, Variant
    from tsgemm.kernels import run_native

    from oracle.rng import uniform_block
    P = Precision.DOUBLE if prec == "double" else Precision.SINGLE
    rows = min(m, 30720 if k > 64 else 1 << 20)
    cols = min(k, 64)
    A = uniform_block(range(rows), range(cols), 1, P.dtype)
    B = uniform_block(range(cols), range(n), 2, P.dtype)
    mA, mB = Matrix.from_2d(A, P), Matrix.from_2d(B, P)
    mC = Matrix.zeros(rows, n, P)
    v = Variant.V3 if k > 64 else Variant.L_OPT2
    params = KernelParams(t1=128, t2=n, t3=4, tcf=1, variant=v)
    t_end, reps, t_tot = time.perf_counter() + budget_s, 0, 0.0
    while reps == 0 or time.perf_counter() < t_end:
        t0 = time.perf_counter()
        run_native(v, mA, mB, mC, params)
        t_tot += time.perf_counter() - t0
        reps += 1
    rate = 2.0 * rows * cols * n * reps / t_tot / 1e9
    return {"value": round(rate, 4), "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"tsgemm.kernels.run_native (baseline/_ref, unmodified) on A[:{rows}, :{cols}] (n={n}, {prec}), "
                      f"{reps} calls, one thread as written (numpy elementwise ops)"}


# ------------------------------------------------------------------------------------------------
def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2002_03258_b200 as tsm
    from paper_2002_03258_b200 import _lib
    from paper_2002_03258_b200.multi import RowShards, broadcast_b, colmajor_buffer

    m_cfg, k, n, prec, variant, c_is_zero, desc, scaling = spec(wl)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    # under torchrun (RANK in the environment) the process group is always created, N=1 included,
    # so the NCCL broadcast path runs at every N. TSM2X_BENCH_SHARE_GPU=1 (test only): all ranks on
    # cuda:0 over gloo, to exercise the multi-rank path on a one-GPU box; not bench values.
    distributed = "RANK" in os.environ
    share = os.environ.get("TSM2X_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = None
    if distributed:
        backend = "gloo" if share else "nccl"
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # the log shows NCCL's rank count and transport
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    dt = torch.float64 if prec == "double" else torch.float32
    eb = 8 if prec == "double" else 4
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev)

    # ---- inputs resident in HBM: this rank's row shard of the (m_total x k) A and (m_total x n) C
    sh = RowShards(scaling, world, rank, m_total=m_cfg, rows_per_rank=m_cfg)
    m, r0 = sh.rows, sh.r0
    A = tsm.colmajor_empty(m, k, dt, dev)
    tsm.fill_uniform(A, seed=1, row_offset=r0)
    B = tsm.colmajor_empty(k, n, dt, dev)
    tsm.fill_uniform(B, seed=2)
    C = tsm.colmajor_empty(m, n, dt, dev)
    if c_is_zero:
        C.zero_()
    else:
        tsm.fill_uniform(C, seed=3, row_offset=r0)
    Bbuf = colmajor_buffer(k, n, dt, dev) if distributed else None
    flush = flush_l2_needed(m, k, eb)
    scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush else None
    red = torch.empty((), dtype=torch.float32, device=dev) if flush else None
    torch.cuda.synchronize()

    def step(kev=None, bev=None):
        if bev is not None:
            bev[0].record(stream)
        Bl = broadcast_b(B if rank == 0 else None, k, n, dt, dev, out=Bbuf) if distributed else B
        if bev is not None:
            bev[1].record(stream)
        if kev is not None:
            lib.tsm2x_set_kernel_events(ctypes.c_void_p(kev[0].cuda_event), ctypes.c_void_p(kev[1].cuda_event))
        tsm.gemm(A, Bl, C, variant=variant, c_is_zero=c_is_zero)

    for _ in range(args.warmup):
        step()
    mk = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))  # noqa: E731
    kevs = [mk() for _ in range(args.steps)]
    bevs = [mk() for _ in range(args.steps)]
    sevs = [mk() for _ in range(args.steps)]
    for pair in kevs + bevs + sevs:  # materialise the CUDA events before handing them to the library
        for e in pair:
            e.record(stream)
    # small problems (L2-flushed workloads) are shorter than the host's enqueue of one call: the
    # step is captured once as a CUDA graph and replayed, so the GPU never waits on Python between
    # the flush and the step. The call-timing events go in a second graph, timed after the timed
    # region under the same flush, so the timed graph holds nothing but the call.
    graph = gtimed = None
    if flush and not distributed:
        gkev = mk()
        for e in gkev:
            e.record(stream)
        cap = torch.cuda.Stream(dev)  # capture needs a side stream; one eager call sizes its workspace
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            step()
        torch.cuda.synchronize()
        graph, gtimed = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            step()
        with torch.cuda.graph(gtimed, stream=cap):
            step(gkev)
        torch.cuda.synchronize()
    t0, t1 = mk()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        if not flush:
            # ~1 ms GPU spin before t0 (outside the timed region): the host enqueues the first steps
            # while the GPU waits on it, so the K timed steps run back to back instead of the first
            # one waiting for Python's first enqueue (a blocking-kernel start, as nvbench does)
            torch.cuda._sleep(2_000_000)
        t0.record(stream)
        for i in range(args.steps):
            if flush:
                torch.sum(scratch, dim=0, out=red)  # 252 MB read: evicts A from the 126 MB L2, leaves it clean
            if flush:  # per-step events only where steps are timed one by one (flush in between)
                sevs[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step(kevs[i], bevs[i] if distributed else None)  # broadcast events only where there is one
            if flush:
                sevs[i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    kern_list = []
    if gtimed is not None:
        for i in range(args.steps):
            torch.sum(scratch, dim=0, out=red)
            gtimed.replay()
            torch.cuda.synchronize()
            kern_list.append(gkev[0].elapsed_time(gkev[1]))
    # launches in the timed region: counted by the library per enqueue; a replayed graph re-runs
    # the launches it captured (counted once at capture)
    launches = _lib.launch_count() - launches0
    if graph is not None:
        launches = graph_launches * args.steps if (graph_launches := _graph_launch_count(step)) else launches
    if distributed:
        dist.barrier()
    # flushed runs: the sum of the per-step events (flush excluded); else the whole timed region
    ms_total = sum(a_.elapsed_time(b_) for a_, b_ in sevs) if flush else t0.elapsed_time(t1)
    kern_ms = (sum(kern_list) if graph is not None else sum(a_.elapsed_time(b_) for a_, b_ in kevs)) / args.steps
    bcast_ms = sum(a_.elapsed_time(b_) for a_, b_ in bevs) / args.steps if distributed else 0.0
    # device idle between consecutive steps (end of step i -> start of step i+1), and from t0 to the
    # first step: evidence that the timed region is the steps back to back
    gaps = [kevs[i][1].elapsed_time(kevs[i + 1][0]) for i in range(args.steps - 1)] if graph is None else []
    step_gap_us = round(1000 * sum(gaps) / len(gaps), 2) if gaps else None
    lead_us = round(1000 * t0.elapsed_time(kevs[0][0]), 2) if graph is None else None
    if distributed:
        t = torch.tensor([ms_total, kern_ms, bcast_ms], device=dev, dtype=torch.float64)
        if backend == "gloo":
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, kern_ms, bcast_ms = float(t[0]), float(t[1]), float(t[2])
    flops_all, byts_all = algorithmic(sh.m_total, k, n, eb, c_is_zero)
    byts_all += (world - 1) * k * n * eb if world > 1 else 0  # every shard reads B once
    _, byts = algorithmic(m, k, n, eb, c_is_zero)  # this rank's kernel
    ms_step = ms_total / args.steps
    value = flops_all / (ms_step * 1e-3) / 1e9
    gbps = byts_all / (ms_step * 1e-3) / 1e9
    peak, peak_src = measured_peaks()
    kern_gbps = byts / (kern_ms * 1e-3) / 1e9
    traffic = ncu_traffic(wl)

    # ---- e2e through the host-buffer C ABI (pinned host buffers), every rank its shard
    e2e = None
    if args.e2e_steps > 0:
        e2e = run_e2e(args, A, B, C, m, k, n, dt, eb, variant, c_is_zero, world, distributed, backend, dev,
                      flops_all)
        if world == 1 and not args.no_drop_in:
            e2e["drop_in"] = run_drop_in(args, A, B, C, m, k, n, prec, variant, c_is_zero, flops_all)

    # ---- CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = host_threads()
        rows, cols = cpu_sample_shape(m, k, args.cpu_elems)
        Ah, Bh, Chh = cpu_sample_inputs(m, k, n, prec, c_is_zero, rows, cols)
        t = min(cpu_time(Ah, Bh, Chh, threads) for _ in range(2))
        rate = 2.0 * rows * cols * n / t / 1e9
        # a strong CPU line beside it: BLAS C + A@B on the same sample — not the
        # reference's path, context for the GPU/CPU ratio only
        tb = []
        for _ in range(3):
            t0_ = time.perf_counter()
            _ = Chh + Ah @ Bh
            tb.append(time.perf_counter() - t0_)
        blas = 2.0 * rows * cols * n / min(tb) / 1e9
        del Ah, Bh, Chh
        cpu = {"value": round(rate, 4), "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"A[:{rows}, :{cols}] of the {m} x {k} A (n={n}, {prec}), best of 2; reference run_native body "
                         f"(kernels.py:391-416) restated in numpy (oracle/reference.py) on {threads} threads",
               "blas_not_reference": {"value": round(blas, 3), "unit": UNIT,
                                      "what": "numpy BLAS C + A@B on the same sample, all threads (not the reference path)"}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64" if prec == "double" else "f32",
            "data": "synthetic: counter-based U[0,1) generated on device (oracle/rng.py regenerates any slab)",
            "config": bench_config(wl, world),
            "timing": ("each step one CUDA-graph replay of the call (captured once), device events around it; "
                       "kernel_ms from a second graph with events around the call" if graph is not None
                       else "device events around the K eagerly enqueued steps"),
            "step_gap_us": step_gap_us, "lead_us": lead_us,
            "GBps": round(gbps, 1),
            "roofline": {"bound": "hbm", "achieved": round(kern_gbps, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(kern_gbps / peak, 4), "traffic": traffic,
                         "kernel": kernel_name(prec, m, k, n, c_is_zero),
                         "kernel_ms": round(kern_ms, 5), "algorithmic_bytes_per_launch": byts,
                         "peak_source": peak_src,
                         "read_stream_ceiling_gbs": 7300.0,
                         "frac_of_read_stream": round(kern_gbps / 7300.0, 4)},
            "comm": ({"backend": backend, "op": "broadcast of B from rank 0 every step", "bytes": k * n * eb,
                      "ms_per_step": round(bcast_ms, 5), "world": world} if distributed else None),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


def _graph_launch_count(step):
    """Library launches one step enqueues (what each replay of its captured graph re-runs)."""
    import torch

    from paper_2002_03258_b200 import _lib
    n0 = _lib.launch_count()
    step()
    torch.cuda.synchronize()
    return _lib.launch_count() - n0


def run_e2e(args, A, B, C, m, k, n, dt, eb, variant, c_is_zero, world, distributed, backend, dev, flops_all):
    """Same metric through tsm2x_run_host (the C-ABI drop-in for run_native) from pinned host
    buffers: every step copies this rank's A shard (and B, C) host->device and C back."""
    import torch
    import torch.distributed as dist

    from paper_2002_03258_b200 import _lib
    from paper_2002_03258_b200.core import Variant
    lib = _lib.load()
    try:
        hA = torch.empty((k, m), dtype=dt, pin_memory=True)  # (k, m) row-major == A column-major, lda=m
        pinned = True
    except Exception:
        hA = torch.empty((k, m), dtype=dt)
        pinned = False
    hA.copy_(A.t())
    hB = B.t().contiguous().cpu().pin_memory()      # (n, k) row-major == B column-major, ldb=k
    hC = torch.empty((n, m), dtype=dt, pin_memory=True)
    hC.copy_(C.t())
    hOut = torch.empty((n, m), dtype=dt, pin_memory=True)
    p = _lib.Params(128, 1, 4, 1, Variant.parse(variant).ordinal)
    flags = _lib.FLAG_C_IS_ZERO if c_is_zero else 0
    precision = _lib.DOUBLE if dt == torch.float64 else _lib.SINGLE

    def call():
        rc = lib.tsm2x_run_host(Variant.parse(variant).ordinal, precision, m, k, n, hA.data_ptr(), m,
                                hB.data_ptr(), k, hC.data_ptr(), hOut.data_ptr(), m, ctypes.byref(p), flags,
                                torch.cuda.current_device())
        _lib.check(rc)

    call()  # warm-up (allocations, staging)
    if distributed:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        call()
    t = (time.perf_counter() - t0) / args.e2e_steps
    if distributed:
        tt = torch.tensor([t], dtype=torch.float64, device="cpu" if backend == "gloo" else dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt[0])
    h2d = eb * (k * m + k * n + (0 if c_is_zero else m * n))
    d2h = eb * m * n
    del hA
    return {"value": round(flops_all / t / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world, "ms_per_step": round(t * 1e3, 3), "steps": args.e2e_steps,
            "host_buffers": "pinned" if pinned else "pageable",
            "api": "tsm2x_run_host (C ABI drop-in for run_native), H2D of A pipelined with the kernels; max over ranks"}


def run_drop_in(args, A, B, C, m, k, n, prec, variant, c_is_zero, flops_all):
    """The reference user's call: paper_2002_03258_b200.run_native(variant, Matrix, Matrix, Matrix,
    KernelParams) on pageable numpy storage (reference kernels.py:391-416). Matrix construction
    (a copy of A, as the reference's Matrix.__init__ makes, core.py:93-106) is timed separately."""
    import numpy as np

    import paper_2002_03258_b200 as tsm
    a_np = A.t().contiguous().cpu().numpy().reshape(-1)  # column-major flat, ld = m
    b_np = B.t().contiguous().cpu().numpy().reshape(-1)
    c_np = np.zeros(m * n, a_np.dtype) if c_is_zero else C.t().contiguous().cpu().numpy().reshape(-1)
    t0 = time.perf_counter()
    Am = tsm.Matrix(m, k, a_np, prec)
    t_construct = time.perf_counter() - t0
    del a_np
    Bm, Cm = tsm.Matrix(k, n, b_np, prec), tsm.Matrix(m, n, c_np, prec)
    params = tsm.KernelParams(t1=128, t2=n, t3=4, tcf=1, variant=tsm.Variant.parse(variant))
    v = tsm.Variant.parse(variant)
    tsm.run_native(v, Am, Bm, Cm, params)  # warm-up (pinned staging buffers, device buffers)
    steps = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(steps):
        out = tsm.run_native(v, Am, Bm, Cm, params)
    t = (time.perf_counter() - t0) / steps
    del out, Am
    eb = 8 if prec == "double" else 4
    return {"value": round(flops_all / t / 1e9, 3), "unit": UNIT, "ms_per_step": round(t * 1e3, 3), "steps": steps,
            "h2d_bytes_per_step": eb * (k * m + k * n + (0 if c_is_zero else m * n)),
            "d2h_bytes_per_step": eb * m * n, "host_buffers": "pageable (numpy Matrix storage)",
            "matrix_construction_ms": round(t_construct * 1e3, 3),
            "value_with_construction": round(flops_all / (t + t_construct) / 1e9, 3),
            "api": "paper_2002_03258_b200.run_native(Variant, Matrix, Matrix, Matrix, KernelParams) -> Matrix"}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="tsm2r_fp64_n8")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-elems", type=int, default=1 << 26, help="elements of A in the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-drop-in", action="store_true", help="skip the run_native (pageable Matrix) e2e leg")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference_arm(args, args.workload)
    else:
        run_ours(args, args.workload)


if __name__ == "__main__":
    main()
