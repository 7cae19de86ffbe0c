#!/usr/bin/env python
"""Benchmark of the fused quantizer hot path on B200 (BASELINE.json metric:
"quantize GB/s vs HBM peak (float/fixed/BFP); quant-GEMM GFLOP/s at 1-8 GPUs").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference          # the reference's CPU path

A step = one pass of the hot path over one batch of synthetic input.  Default
workload (BASELINE.json configs[1], the config the metric is quoted on):
fixed-point wl=8 fl=4 saturating, stochastic rounding, over a 2^30-element
fp32 tensor per GPU.  At N GPUs each rank owns a 2^30-element shard of a
global N*2^30 tensor (flat-index RNG offsets, no collective on the data
path): weak scaling.  Other configs (--config c1/c3/c4) are reported the same
way for DESIGN.md; c2 is the driver's line.

value     : algorithmic bytes (read + write, 8 B/element) of all ranks per
            second, inputs resident in HBM (device-generated with the
            reference's own random_uniform, bit-identical), CUDA events on the
            launching stream, max over ranks.
e2e       : the same metric through the host entry point lpq_quantize_host
            (pinned host buffers; H2D + kernels + D2H inside the timed region).
roofline  : the quantize kernel's algorithmic bytes / its mean CUDA-event
            duration vs the measured HBM copy peak (MEASURED_PEAKS.json).
cpu_baseline: the reference library (oracle/_ref, compiled from the
            reference sources) timed on this host's cores on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GIB = 1 << 30
SEED = 0x15EED  # proj/src/bench.cpp:56


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)", {}


def load_traffic(kernel_key):
    """dram bytes per launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        return d.get(kernel_key)
    except Exception:
        return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    5 ms on a side thread DURING the timed region (nvidia-smi's own sampling
    starts too slowly for millisecond regions)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, local_rank):
        self.local_rank = local_rank
        self.samples = []
        self.stop = threading.Event()
        self.h = None
        self.max_mhz = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = self.local_rank
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.local_rank < len(ids):
                tok = ids[self.local_rank]
                if tok.isdigit():
                    idx = int(tok)
                else:
                    return pynvml.nvmlDeviceGetHandleByUUID(tok)
        return pynvml.nvmlDeviceGetHandleByIndex(idx)

    def _sample(self):
        import pynvml
        sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        try:
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((sm, r))

    def _run(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.005)

    def __enter__(self):
        try:
            import pynvml
            self.h = self._handle()
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:
            self.h = None
            self.err = str(e)
        return self

    def __exit__(self, *exc):
        if self.h is not None:
            try:
                self._sample()  # one sample at the end of the region
            except Exception:
                pass
            self.stop.set()
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [],
                    "samples": 0, "source": getattr(self, "err", "nvml")}
        reasons = set()
        for _, r in self.samples:
            for bit, name in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s for s, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------------------
def cpu_reference_time(fmt_c, mode, xs, shape, threads, repeats):
    """Median wall time of the reference's quantize_fused_at on the host."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import RefLib
    ref = RefLib()
    ref.set_num_threads(threads)
    xs = xs.reshape(shape)
    times = []
    ref.quantize(xs, fmt_c, mode, seed=SEED, call=0, timed=True)  # warmup
    for _ in range(repeats):
        st, y, secs = ref.quantize(xs, fmt_c, mode, seed=SEED, call=0, timed=True)
        assert st == 0
        times.append(secs)
    return statistics.median(times)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
CONFIGS = {
    "c1": dict(workload="C1: float exp=5 man=2 (FP8-like), stochastic rounding, "
                        "2^24-element fp32 tensor per GPU (rotating buffers > L2)",
               kind="float", n=1 << 24, fmt=("float", 5, 2), mode="stochastic"),
    "c1n": dict(workload="C1: float exp=5 man=2, nearest-even, 2^24 elements per GPU "
                         "(rotating buffers > L2)",
                kind="float", n=1 << 24, fmt=("float", 5, 2), mode="nearest_even"),
    "c1log": dict(workload="C1 log-uniform variant (SURVEY 8(d)): float exp=5 man=2, "
                           "stochastic, 2^24 elements with |x| log-uniform in "
                           "[2^-20, 2^20] and random sign (underflow and saturation "
                           "branches; rotating buffers > L2)",
                  kind="float", n=1 << 24, fmt=("float", 5, 2), mode="stochastic",
                  dist="loguniform"),
    "c1logn": dict(workload="C1 log-uniform variant: float exp=5 man=2, nearest-even, "
                            "2^24 elements, |x| log-uniform in [2^-20, 2^20]",
                   kind="float", n=1 << 24, fmt=("float", 5, 2), mode="nearest_even",
                   dist="loguniform"),
    "c1big": dict(workload="float exp=5 man=2, stochastic, 2^30 elements (diagnostic)",
                  kind="float", n=1 << 30, fmt=("float", 5, 2), mode="stochastic"),
    "c2": dict(workload="C2: fixed-point wl=8 fl=4 saturating, stochastic rounding, "
                        "2^30-element fp32 tensor per GPU",
               kind="fixed", n=1 << 30, fmt=("fixed", 8, 4), mode="stochastic"),
    "c3": dict(workload="C3: block floating point wl=8, shared exponent per row of a "
                        "65536x4096 fp32 matrix per GPU, nearest-even",
               kind="block", n=1 << 28, rows=65536, cols=4096, fmt=("block", 8, 0),
               mode="nearest_even"),
    "c3s": dict(workload="C3: block wl=8 per row of 65536x4096, stochastic",
                kind="block", n=1 << 28, rows=65536, cols=4096, fmt=("block", 8, 0),
                mode="stochastic"),
}


def make_spec(q, cfg):
    kind, a, b = cfg["fmt"]
    if kind == "float":
        f = q.FloatFormat(a, b)
    elif kind == "fixed":
        f = q.FixedFormat(a, b)
    else:
        f = q.BlockFloatFormat(a, b)
    mode = {"stochastic": q.RoundingMode.Stochastic,
            "nearest_even": q.RoundingMode.NearestEven}[cfg["mode"]]
    return q.QuantSpec(f, mode, SEED, 0)


def oracle_fmt(cfg):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import block_fmt, fixed_fmt, float_fmt
    kind, a, b = cfg["fmt"]
    return {"float": float_fmt, "fixed": fixed_fmt}[kind](a, b) if kind != "block" \
        else block_fmt(a, b)


def mode_id(cfg):
    return {"stochastic": 0, "nearest_even": 1}[cfg["mode"]]


def make_input(q, cfg, shape, i, dev, base):
    """Synthetic input of SURVEY §8(d), generated on the device with the
    reference's own random_uniform (tensor.cpp:430-440, bit-identical), buffer
    i of the rotating set (i = 0 is the workload's tensor itself):
      C1 : random_uniform(RngStream{7}, call i, -4, 4)  (bench.cpp:58-60)
      C2 : random_uniform(RngStream{2}, call i, -10, 10)
      C3 : random_uniform(RngStream{3}, call i, -1, 1) x 2^s_r per row, s_r an
           integer uniform in [-20, 20] (random_uniform(RngStream{4}) of the row)
      log-uniform C1 variant: |x| = 2^U(-20, 20), random sign."""
    import torch
    if cfg.get("dist") == "loguniform":  # |x| = 2^U(-20, 20), random sign
        return torch.copysign(
            torch.exp2(q.random_uniform(shape, 50, i, -20.0, 20.0, device=dev, index_base=base)),
            q.random_uniform(shape, 60, i, -1.0, 1.0, device=dev, index_base=base))
    if cfg["kind"] == "float":
        return q.random_uniform(shape, 7, i, -4.0, 4.0, device=dev, index_base=base)
    if cfg["kind"] == "block":
        rows = shape[0]
        x = q.random_uniform(shape, 3, i, -1.0, 1.0, device=dev, index_base=base)
        r0 = base // shape[1]
        s = torch.floor(q.random_uniform((rows, 1), 4, i, -20.0, 21.0, device=dev,
                                         index_base=r0)).clamp_(-20, 20)
        return x * torch.exp2(s)
    return q.random_uniform(shape, 2, i, -10.0, 10.0, device=dev, index_base=base)


def host_input(cfg, shape):
    """make_input(buffer 0) through the reference library on the host (the
    --impl reference arm; same values bit for bit)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import RefLib
    ref = RefLib()
    if cfg.get("dist") == "loguniform":
        u = ref.random_uniform(shape, 50, 0, -20.0, 20.0)
        sg = ref.random_uniform(shape, 60, 0, -1.0, 1.0)
        return np.copysign(np.exp2(u), sg).astype(np.float32)
    if cfg["kind"] == "float":
        return ref.random_uniform(shape, 7, 0, -4.0, 4.0)
    if cfg["kind"] == "block":
        x = ref.random_uniform(shape, 3, 0, -1.0, 1.0)
        s = np.clip(np.floor(ref.random_uniform((shape[0], 1), 4, 0, -20.0, 21.0)), -20, 20)
        x *= np.exp2(s).astype(np.float32)
        return x
    return ref.random_uniform(shape, 2, 0, -10.0, 10.0)


# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import ctypes as C
    import paper_1910_04540_b200 as q
    from paper_1910_04540_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = CONFIGS[args.config]
    spec = make_spec(q, cfg)
    n = cfg["n"]
    shape = (cfg["rows"], cfg["cols"]) if cfg["kind"] == "block" else (n,)
    base = rank * n  # global flat index of this shard
    # input generated on the device, bit-identical to the reference generator
    nbuf = 1
    if n * 4 * 2 < 512 << 20:  # small config: rotate buffers so L2 cannot hold them
        nbuf = max(2, (512 << 20) // (n * 8))
    xs = [make_input(q, cfg, shape, i, dev, base) for i in range(nbuf)]
    ys = [torch.empty_like(x) for x in xs]
    stream = torch.cuda.current_stream(dev)
    status = q.quant._status_buf(dev)
    fmt_c = spec.format.c()
    shp = _lib.shape_array(shape)
    wsb = _lib.lib.lpq_workspace_size(C.byref(fmt_c), shp, len(shape))
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
    sptr = C.c_void_p(stream.cuda_stream)

    def step(i, sp=sptr):
        x, y = xs[i % nbuf], ys[i % nbuf]
        st = _lib.lib.lpq_quantize(
            C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), shp, len(shape),
            base, C.byref(fmt_c), int(spec.mode), SEED, 0,
            C.c_void_p(ws.data_ptr()), wsb, C.c_void_p(status.data_ptr()), sp)
        _lib.check(st, "quantize")

    for i in range(args.warmup):
        step(i)
    _lib.check(_lib.lib.lpq_status_fetch(C.c_void_p(status.data_ptr()), sptr))
    # launch-bound configs (a step shorter than the host's per-call Python +
    # ctypes overhead): the K timed steps are captured into ONE CUDA graph
    # and replayed once, so the device is never starved by the host; the
    # per-launch duration is then the graph time / K (kernels back to back)
    use_graph = args.graph == "on" or (args.graph == "auto" and 8 * n < (1 << 30))
    graph = None
    launches0 = q.launch_count()
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                for i in range(args.steps):
                    step(i, C.c_void_p(side.cuda_stream))
        stream.wait_stream(side)
        captured = q.launch_count()
        graph.replay()  # untimed: uploads the graph
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if not use_graph:
        launches0 = q.launch_count()
    with ClockSampler(local_rank) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        if use_graph:
            graph.replay()
        else:
            for i in range(args.steps):
                ev[i][0].record(stream)
                step(i)
                ev[i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    launches = (captured if use_graph else q.launch_count()) - launches0
    _lib.check(_lib.lib.lpq_status_fetch(C.c_void_p(status.data_ptr()), sptr))
    elapsed = t0.elapsed_time(t1) / 1e3
    kern = ([elapsed / args.steps] * args.steps if use_graph
            else [a.elapsed_time(b) / 1e3 for a, b in ev])
    if world > 1:
        t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        dist.barrier()
    bytes_per_rank_step = 8 * n
    value = bytes_per_rank_step * world * args.steps / elapsed / 1e9
    # ---- e2e through the host entry point (pinned host buffers) -----------------
    e2e = None
    if not args.no_e2e:
        host_mem = "pinned"
        try:
            hx = torch.empty(shape, dtype=torch.float32, pin_memory=True)
            hy = torch.empty(shape, dtype=torch.float32, pin_memory=True)
        except RuntimeError:  # not enough page-lockable memory: pageable path
            host_mem = "pageable"
            hx = torch.empty(shape, dtype=torch.float32)
            hy = torch.empty(shape, dtype=torch.float32)
        hx.copy_(xs[0])
        e_steps = max(1, min(args.steps, args.e2e_steps))

        def hstep():
            st = _lib.lib.lpq_quantize_host(
                C.c_void_p(hx.data_ptr()), C.c_void_p(hy.data_ptr()), shp,
                len(shape), base, C.byref(fmt_c), int(spec.mode), SEED, 0,
                local_rank)
            _lib.check(st, "quantize_host")
        hstep()  # warm the context (pinned staging, streams)
        if world > 1:
            dist.barrier()
        tt = time.perf_counter()
        for _ in range(e_steps):
            hstep()
        et = time.perf_counter() - tt
        if world > 1:
            t = torch.tensor([et], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        # the host result must equal the device result
        assert torch.equal(hy.view(torch.int32), ys[0].cpu().view(torch.int32))
        # the PCIe ceiling for the same bytes: a bare H2D of the input concurrent
        # with a bare D2H of the output (two streams, same host buffers), no
        # kernel -- what the e2e number is bounded by
        ceiling = None
        if host_mem == "pinned":
            dtmp = torch.empty_like(xs[0])
            s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            ct = []
            for _ in range(3):
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                with torch.cuda.stream(s_in):
                    dtmp.copy_(hx, non_blocking=True)
                with torch.cuda.stream(s_out):
                    hy.copy_(ys[0], non_blocking=True)
                torch.cuda.synchronize(dev)
                ct.append(time.perf_counter() - t0)
            ceiling = round(bytes_per_rank_step / min(ct) / 1e9, 3)
            del dtmp
        b_in, b_out = C.c_int(), C.c_int()
        _lib.lib.lpq_host_bytes_per_element(C.byref(fmt_c), int(spec.mode), C.byref(b_in),
                                            C.byref(b_out))
        e2e = {"value": round(bytes_per_rank_step * world * e_steps / et / 1e9, 3),
               "unit": "GB/s", "h2d_bytes_per_step": b_in.value * n * world,
               "d2h_bytes_per_step": b_out.value * n * world, "steps": e_steps,
               "api": f"lpq_quantize_host (include/lpq.h), {host_mem} host buffers",
               "pcie_copy_ceiling": ceiling,
               "pcie_copy_ceiling_note": "per GPU: concurrent bare H2D(input)+D2H(output) fp32 "
                                         "copies of the same pinned buffers, metric units",
               "d2h_format": ("one-byte codes of the quantized values, decoded on the host "
                              "(bit-identical; include/lpq.h)" if b_out.value == 1
                              else "fp32")}
        del hx, hy
    # ---- roofline of the dominant kernel --------------------------------------------
    peak, peak_src, peaks = load_peaks()
    # context for the peak: a plain device-to-device copy of the same buffers
    # (torch copy_, the driver's own peak probe) measured in this process
    cps = []
    for _ in range(3):
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        ys[0].copy_(xs[0])
        c1.record(stream)
        torch.cuda.synchronize()
        cps.append(c0.elapsed_time(c1) / 1e3)
    copy_gbs = 8 * n / min(cps) / 1e9
    kmean = statistics.mean(kern)
    achieved = bytes_per_rank_step / kmean / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4),
            "traffic": load_traffic(args.config), "peak_source": peak_src,
            "algorithmic_bytes_per_launch": bytes_per_rank_step,
            "kernel_ms_mean": round(kmean * 1e3, 4),
            "kernel_ms_min": round(min(kern) * 1e3, 4),
            "kernel_time_source": ("CUDA-graph replay of the K launches / K (back to back)"
                                   if use_graph else "CUDA events around each launch"),
            "frac_of_8TBs_spec": round(achieved / 8000.0, 4),
            "d2d_copy_same_buffers_gbs": round(copy_gbs, 1)}
    # ---- CPU baseline (rank 0, N = 1 only) ------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            samp = min(n, args.cpu_sample)
            if cfg["kind"] == "block":
                samp_shape = (samp // cfg["cols"], cfg["cols"])
            else:
                samp_shape = (samp,)
            xh = xs[0].reshape(-1)[:samp].cpu().numpy()
            th = cpu_threads()
            secs = cpu_reference_time(oracle_fmt(cfg), mode_id(cfg), xh, samp_shape,
                                      th, args.cpu_repeats)
            # one thread too, on a quarter of the sample
            s1 = samp // 4 if cfg["kind"] != "block" else (samp // 4 // cfg["cols"]) * cfg["cols"]
            s1_shape = (s1 // cfg["cols"], cfg["cols"]) if cfg["kind"] == "block" else (s1,)
            secs1 = cpu_reference_time(oracle_fmt(cfg), mode_id(cfg), xh[:s1], s1_shape, 1, 1)
            cpu = {"value": round(8 * samp / secs / 1e9, 4), "unit": "GB/s",
                   "cores": th, "kind": "reference",
                   "sample": f"first {samp} elements of this workload's input, "
                             f"lpsim::quantize_fused_at (oracle/_ref, -O3), "
                             f"set_num_threads({th}), median of {args.cpu_repeats}",
                   "value_1thread": round(8 * s1 / secs1 / 1e9, 4),
                   "cpu_model": cpu_model()}
        except Exception as e:  # the baseline must not sink the GPU line
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    out = {
        "metric": "quantize GB/s vs HBM peak (float/fixed/BFP); quant-GEMM GFLOP/s at 1-8 GPUs",
        "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(elapsed / args.steps * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32 (u32/fp32 bit arithmetic)", "data": "synthetic (device-side "
        "random_uniform, bit-identical to the reference generator)",
        "config": {"workload": cfg["workload"], "elements_per_gpu": n,
                   "format": "%s:%d:%d" % cfg["fmt"], "rounding": cfg["mode"],
                   "global_elements": n * world, "parallelism": f"shard{world}",
                   "l2": ("inputs larger than L2" if nbuf == 1 else
                          f"{nbuf} rotating input/output buffers, "
                          f"{nbuf * n * 8 >> 20} MiB > 126 MB L2"),
                   "launch": ("the K timed steps captured in one CUDA graph (launch-bound "
                              "from Python otherwise)" if use_graph else "stream launches")},
        "e2e": e2e, "gpu_launches": launches, "roofline": roof,
        "cpu_baseline": cpu, "clocks": clk.summary(),
    }
    return out


# ---------------------------------------------------------------------------
def run_gemm(args, rank, world, local_rank):
    """C4: per-op-rounded GEMM 4096^3, float(8,7) after every multiply and add.
    c4: operands quantized to float(8,7) first, nearest rounding (the
    hardware-bf16 kernel); c4raw: raw fp32 operands (the FMUL + cvt.rn.bf16x2
    kernel); c4s: stochastic rounding after every op (the general kernel)."""
    import torch
    import torch.distributed as dist
    import paper_1910_04540_b200 as q
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_1910_04540_b200.shard import broadcast_operand, gemm_rows
    M = N = K = 4096
    # the BASELINE problem (4096^3) split by output rows over the ranks
    # (strong scaling): rank r owns rows [lo, hi) of A and C, passes
    # row_base = lo (global variate index), and B is generated once on rank 0
    # and broadcast, outside the timed region
    lo, hi = gemm_rows(M, rank, world)
    f87 = q.QuantSpec(q.FloatFormat(8, 7))
    raw = args.config == "c4raw"
    mode = q.RoundingMode.Stochastic if args.config == "c4s" else q.RoundingMode.NearestEven
    prep = (lambda t: t) if raw else (lambda t: q.quantize_fused_at(t, f87, 0))
    a = prep(q.random_uniform((hi - lo, K), 41, 0, -1.0, 1.0, device=dev, index_base=lo * K))
    if rank == 0:
        b = prep(q.random_uniform((K, N), 42, 0, -1.0, 1.0, device=dev))
    else:
        b = torch.empty((K, N), device=dev)
    broadcast_operand(b)
    c = torch.empty((hi - lo, N), device=dev)
    fm = q.FloatFormat(8, 7)
    for _ in range(args.warmup):
        q.quant_gemm(a, b, fm, fm, mode, 0x5EED, 0, out=c, sync=False, row_base=lo)
    q.fetch_status(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = q.launch_count()
    s = torch.cuda.current_stream(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        t0.record(s)
        for _ in range(args.steps):
            q.quant_gemm(a, b, fm, fm, mode, 0x5EED, 0, out=c, sync=False, row_base=lo)
        t1.record(s)
        torch.cuda.synchronize()
    q.fetch_status(dev)
    el = t0.elapsed_time(t1) / 1e3
    if world > 1:
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    flops = 2.0 * M * N * K  # the whole problem, all ranks
    value = flops * args.steps / el / 1e9
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_t = sms * 128 * 2 * 1.965e9 / 1e12
    ach = flops * args.steps / el / 1e12 / world  # per GPU
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the per-op GEMM is not in the reference: its restatement (oracle/,
        # the definition the tests check against), rows split over the host
        # threads (ctypes releases the GIL), on a sample of output rows
        try:
            import time as _t
            from concurrent.futures import ThreadPoolExecutor
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from oracle_lib import Oracle, float_fmt
            o = Oracle()
            th = cpu_threads()
            rows = 2 * th
            ah = a[:rows].cpu().numpy()
            bh = b.cpu().numpy()
            f87o = float_fmt(8, 7)
            t_0 = _t.perf_counter()
            with ThreadPoolExecutor(th) as ex:
                list(ex.map(lambda r: o.quant_gemm(ah[r:r + 2], bh, f87o, f87o, int(mode),
                                                   seed=0x5EED, call=0, row_base=r),
                            range(0, rows, 2)))
            secs = _t.perf_counter() - t_0
            cpu = {"value": round(2.0 * rows * N * K / secs / 1e9, 4), "unit": "GFLOP/s",
                   "cores": th, "kind": "port",
                   "sample": f"{rows} output rows of the 4096^3 problem through the restated "
                             f"per-op GEMM (oracle/lpq_oracle.c; the reference has none), "
                             f"{th} threads", "cpu_model": cpu_model()}
        except Exception as e:  # the baseline must not sink the GPU line
            cpu = {"value": None, "unit": "GFLOP/s", "cores": None, "kind": "port",
                   "sample": f"unavailable: {e}"}
    return {
        "metric": "quant-GEMM GFLOP/s (per-op rounded, float(8,7) after every multiply and add)",
        "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32 ops + bf16 rounding",
        "data": "synthetic", "config": {"workload": "C4: 4096x4096x4096, output rows split "
                                                    "over the GPUs, B broadcast from rank 0" + {
                                            "c4": "; float(8,7) operands, nearest",
                                            "c4raw": "; raw fp32 operands, nearest",
                                            "c4s": "; float(8,7) operands, stochastic after "
                                                   "every op"}[args.config],
                                        "rows_per_gpu": hi - lo,
                                        "parallelism": f"rows{world}"},
        "gpu_launches": q.launch_count() - l0,
        "roofline": {"bound": "fp32_cuda_core", "achieved": round(ach, 2),
                     "peak": round(peak_t, 2), "unit": "TFLOP/s",
                     "frac": round(ach / peak_t, 4), "traffic": load_traffic(args.config),
                     "peak_source": f"{sms} SMs x 128 FP32 lanes x 2 x 1965 MHz",
                     # the bf16 kernels' own bound: an HMUL2/HADD2 (or FMUL
                     # pair + HADD2) per 64 MACs per warp holds the FMA pipe
                     # for 4 cycles -> 16 MAC/clk/SMSP (profiles/r02_pipes.md)
                     "ceiling": None if args.config == "c4s" else {
                         "value": round(sms * 4 * 16 * 2 * 1.965e9 / 1e12, 2),
                         "unit": "TFLOP/s", "frac": round(ach / (sms * 4 * 16 * 2 * 1.965e9 / 1e12), 4),
                         "what": "bf16x2 FMA-pipe issue bound (HMUL2 + HADD2 per 2 MACs)"}},
        "cpu_baseline": cpu, "clocks": clk.summary(),
    }


# ---------------------------------------------------------------------------
FP64_DMMA_PEAK = 37.1  # TFLOP/s, scripts/dmma_rate.cu on the round-1 B200


def run_matmul_q(args, rank, world, local_rank):
    """The reference's quantized_matmul (quant_ops.cpp:191-193) at 4096^3:
    double-accumulated matmul in ascending k with fixed(8,4) stochastic
    quantization fused into the epilogue (lpq_matmul_q, DFMA)."""
    import torch
    import torch.distributed as dist
    import paper_1910_04540_b200 as q
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    M = N = K = 4096
    a = q.random_uniform((M, K), 41, 0, -1.0, 1.0, device=dev, index_base=rank * M * K)
    b = q.random_uniform((K, N), 42, 0, -1.0, 1.0, device=dev)
    c = torch.empty((M, N), device=dev)
    spec = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic, SEED)
    for _ in range(args.warmup):
        q.quantized_matmul_at(a, b, spec, 0, out=c, sync=False, row_base=rank * M)
    q.fetch_status(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = q.launch_count()
    with ClockSampler(local_rank) as clk:
        t0.record(s)
        for _ in range(args.steps):
            q.quantized_matmul_at(a, b, spec, 0, out=c, sync=False, row_base=rank * M)
        t1.record(s)
        torch.cuda.synchronize()
    q.fetch_status(dev)
    el = t0.elapsed_time(t1) / 1e3
    if world > 1:
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    flops = 2.0 * M * N * K
    ach = flops * args.steps / el / 1e12
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference's own quantized_matmul (oracle/_ref) on 32 rows of
        # the problem (its matmul runs serially below m = 4096)
        try:
            import time as _t
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from oracle_lib import RefLib, fixed_fmt
            ref = RefLib()
            ref.set_num_threads(cpu_threads())
            rows = 32
            ah = a[:rows].cpu().numpy()
            bh = b.cpu().numpy()
            t_0 = _t.perf_counter()
            ref.quantized_matmul(ah, bh, fixed_fmt(8, 4), 0, seed=SEED, call=0)
            secs = _t.perf_counter() - t_0
            cpu = {"value": round(2.0 * rows * N * K / secs / 1e9, 4), "unit": "GFLOP/s",
                   "cores": 1, "kind": "reference",
                   "sample": f"lpsim::quantized_matmul on {rows} rows x 4096 x 4096 "
                             f"(oracle/_ref; serial below m = 4096)", "cpu_model": cpu_model()}
        except Exception as e:
            cpu = {"value": None, "unit": "GFLOP/s", "cores": None, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    return {
        "metric": "reference quantized_matmul GFLOP/s (double accumulation, fused quantize epilogue)",
        "value": round(flops * world * args.steps / el / 1e9, 1), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp64 accumulate, fp32 I/O",
        "data": "synthetic", "config": {"workload": "quantized_matmul 4096^3, fixed(8,4) stochastic",
                                        "parallelism": f"shard{world}"},
        "gpu_launches": q.launch_count() - l0,
        "roofline": {"bound": "fp64 tensor (DMMA)", "achieved": round(ach, 2), "unit": "TFLOP/s",
                     "peak": FP64_DMMA_PEAK, "frac": round(ach / FP64_DMMA_PEAK, 4),
                     "traffic": load_traffic("c4ref"),
                     "peak_source": "measured in-repo: register-resident DMMA m8n8k4 loop on "
                                    "this B200 (scripts/dmma_rate.cu; DFMA: 33.4); "
                                    "MEASURED_PEAKS.json has no FP64 figure"},
        "cpu_baseline": cpu, "clocks": clk.summary(),
    }


# ---------------------------------------------------------------------------
def run_sweep(args, rank, world, local_rank):
    """C5: ResNet-50 training-step quantization sweep (batch 256): the 54
    weight, 54 weight-gradient and 54 activation tensors, each through
    float(5,2), fixed(8,4) and block(8, dim 0) (per output channel for
    weights and gradients, per sample for activations); nearest-even for
    weights and activations, stochastic for gradients.  One step = the whole
    sweep (486 quantizations), captured once as a CUDA graph and replayed.
    At N GPUs the sweep's work units are bin-packed over the ranks by bytes
    (shard.binpack; strong scaling: the job is one sweep)."""
    import torch
    import torch.distributed as dist
    import ctypes as C
    import paper_1910_04540_b200 as q
    from paper_1910_04540_b200.resnet50 import ResNet50Sweep
    from paper_1910_04540_b200.shard import binpack

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    mine = binpack(ResNet50Sweep.unit_bytes(256), world)[rank]
    plan = ResNet50Sweep(q, dev, units=mine)
    layers = plan.layers
    tensors = list(plan.inputs.values())
    s0 = torch.cuda.current_stream(dev)
    q.reset_pass_count()
    nbytes = plan.measure_once(C.c_void_p(s0.cuda_stream))
    launches_per_sweep = plan.launches
    calls = [None] * (3 * len(tensors))
    nbytes_all = torch.tensor([float(nbytes)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(nbytes_all)
    nbytes_all = int(nbytes_all.item())
    q.fetch_status(dev)

    def sweep(stream):
        plan.launch(C.c_void_p(stream.cuda_stream))

    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(dev)
    side.wait_stream(s0)
    with torch.cuda.stream(side):
        sweep(side)  # warm the side stream
    s0.wait_stream(side)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=side):
        sweep(side)
    for _ in range(args.warmup):
        g.replay()
    torch.cuda.synchronize()
    q.fetch_status(dev)
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        t0.record(s0)
        for _ in range(args.steps):
            g.replay()
        t1.record(s0)
        torch.cuda.synchronize()
    q.fetch_status(dev)
    el = t0.elapsed_time(t1) / 1e3
    if world > 1:
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    peak, peak_src, _ = load_peaks()
    ach = nbytes * args.steps / el / 1e9  # this rank's share over the job time
    value = nbytes_all * args.steps / el / 1e9
    total_elems = sum(t.numel() for t in tensors)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference's quantize_fused_at on a bounded sample of the sweep:
        # 20 per-sample rows of the first activation ([20, 802816] = 16M
        # floats) through the three formats, all host threads
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from oracle_lib import block_fmt, fixed_fmt, float_fmt
            th = cpu_threads()
            act = q.random_uniform(layers[0][2], 300, 0, -4.0, 4.0, device=dev)
            xh = act.reshape(act.shape[0], -1)[:20].contiguous().cpu().numpy()
            secs = 0.0
            for fo in (float_fmt(5, 2), fixed_fmt(8, 4), block_fmt(8, 0)):
                secs += cpu_reference_time(fo, 1, xh.reshape(-1), xh.shape, th, 1)
            cpu = {"value": round(3 * 8 * xh.size / secs / 1e9, 4), "unit": "GB/s",
                   "cores": th, "kind": "reference",
                   "sample": f"lpsim::quantize_fused_at, nearest, float(5,2) + fixed(8,4) + "
                             f"block(8, dim0) on {xh.shape} of the first activation, "
                             f"{th} threads", "cpu_model": cpu_model()}
        except Exception as e:
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    return {
        "metric": "quantize GB/s vs HBM peak (float/fixed/BFP); quant-GEMM GFLOP/s at 1-8 GPUs",
        "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32 (u32/fp32 bit arithmetic)",
        "data": "synthetic ResNet-50-shaped tensors (no weights available offline)",
        "config": {"workload": "C5: ResNet-50 (batch 256) weights, weight gradients and "
                               "activations through float(5,2), fixed(8,4), block(8, dim0)",
                   "tensors_this_rank": len(tensors),
                   "quantizations_per_step_this_rank": len(calls),
                   "elements_per_sweep_pass_this_rank": total_elems,
                   "algorithmic_bytes_per_step": nbytes_all,
                   "launches_per_step_this_rank": launches_per_sweep,
                   "parallelism": f"binpack{world} (units: weights, gradients, each "
                                  f"activation; by bytes, shard.binpack)"},
        "gpu_launches": launches_per_sweep * args.steps,
        "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(ach / peak, 4), "traffic": None,
                     "peak_source": peak_src},
        "cpu_baseline": cpu, "clocks": clk.summary(),
    }


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref: lpsim compiled unmodified from /root/reference) on the
    host cores with every host thread, same config / metric / unit as our arm.
    Rank 0 only (the other ranks exit without work).

    c1*, c2, c3*: the WHOLE workload per step (same input, bit-identical
    generator): lpsim::quantize_fused_at.  c4ref: lpsim::quantized_matmul on a
    bounded row sample of the 4096^3 problem.  c4: the reference has no
    per-op-rounded GEMM; its restatement (oracle/, the definition the tests
    check against) on a row sample, kind "port".  c5: quantize_fused_at of a
    bounded sample of the sweep (the first activation's rows, three formats)."""
    if rank != 0:
        return None
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import RefLib
    if not RefLib.available():
        return {"impl": "reference", "unavailable": "oracle/_ref/liblpsim_ref.so not built"}
    ref = RefLib()
    th = cpu_threads()
    ref.set_num_threads(th)
    metric = "quantize GB/s vs HBM peak (float/fixed/BFP); quant-GEMM GFLOP/s at 1-8 GPUs"
    kind = "reference"
    same = True
    if args.config in CONFIGS:
        cfg = CONFIGS[args.config]
        n = cfg["n"]
        shape = (cfg["rows"], cfg["cols"]) if cfg["kind"] == "block" else (n,)
        x = host_input(cfg, shape)
        fmt = oracle_fmt(cfg)

        def one():
            st, y, secs = ref.quantize(x, fmt, mode_id(cfg), seed=SEED, call=0, timed=True)
            assert st == 0
            return secs
        per_step, unit = 8 * n, "GB/s"
        sample = (f"the whole workload ({n} elements) per step, lpsim::quantize_fused_at "
                  f"(incl. its output allocation), set_num_threads({th})")
        config = {"workload": cfg["workload"], "elements_per_gpu": n,
                  "format": "%s:%d:%d" % cfg["fmt"], "rounding": cfg["mode"],
                  "parallelism": "host threads"}
    elif args.config in ("c4", "c4raw", "c4s", "c4ref"):
        from oracle_lib import Oracle, fixed_fmt, float_fmt
        from concurrent.futures import ThreadPoolExecutor
        rows = 2 * th if args.config != "c4ref" else 32
        a = ref.random_uniform((rows, 4096), 41, 0, -1.0, 1.0)
        b = ref.random_uniform((4096, 4096), 42, 0, -1.0, 1.0)
        if args.config != "c4ref":
            o = Oracle()
            f87 = float_fmt(8, 7)
            gmode = 0 if args.config == "c4s" else 1
            if args.config != "c4raw":
                _, a = ref.quantize(a, f87, 1)
                _, b = ref.quantize(b, f87, 1)
            kind = "port"

            def one():
                t0 = time.perf_counter()
                with ThreadPoolExecutor(th) as ex:
                    list(ex.map(lambda r: o.quant_gemm(a[r:r + 2], b, f87, f87, gmode,
                                                       seed=0x5EED, call=0, row_base=r),
                                range(0, rows, 2)))
                return time.perf_counter() - t0
            sample = (f"{rows} of the 4096 output rows per step through the restated per-op "
                      f"GEMM (oracle/lpq_oracle.c; the reference has none), {th} threads")
            metric = "quant-GEMM GFLOP/s (per-op rounded, float(8,7) after every multiply and add)"
        else:
            def one():
                t0 = time.perf_counter()
                ref.quantized_matmul(a, b, fixed_fmt(8, 4), 0, seed=SEED, call=0)
                return time.perf_counter() - t0
            sample = (f"lpsim::quantized_matmul on {rows} of the 4096 rows per step "
                      f"(serial below m = 4096)")
            metric = "reference quantized_matmul GFLOP/s (double accumulation, fused quantize epilogue)"
        per_step, unit, same = 2.0 * rows * 4096 * 4096, "GFLOP/s", False
        config = {"workload": f"{args.config}: 4096x4096x4096 (row sample)",
                  "parallelism": "host threads"}
    elif args.config == "c5":
        from oracle_lib import block_fmt, fixed_fmt, float_fmt
        x = ref.random_uniform((20, 802816), 300, 0, -4.0, 4.0)
        fmts = (float_fmt(5, 2), fixed_fmt(8, 4), block_fmt(8, 0))

        def one():
            t = 0.0
            for fo in fmts:
                t += ref.quantize(x, fo, 1, seed=SEED, call=0, timed=True)[2]
            return t
        per_step, unit, same = 3 * 8 * x.size, "GB/s", False
        sample = (f"lpsim::quantize_fused_at, nearest, float(5,2) + fixed(8,4) + block(8, dim0) "
                  f"on {x.shape} per-sample rows of the first ResNet-50 activation, {th} threads")
        config = {"workload": "C5: ResNet-50 sweep (sample)", "parallelism": "host threads"}
    else:
        raise SystemExit(f"--impl reference: unknown config {args.config}")
    for _ in range(args.warmup):
        one()
    times = [one() for _ in range(args.steps)]
    tot = sum(times)
    value = per_step * args.steps / tot / 1e9
    out = {
        "impl": "reference", "metric": metric,
        "value": round(value, 4), "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp64 (reference arithmetic)",
        "data": "synthetic (reference random_uniform)", "config": config,
        "same_work_per_step": same,
        "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": th,
                         "kind": kind, "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    return out


def free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (one rank each); default: WORLD_SIZE under torchrun, else 1")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS) + ["c4", "c4raw", "c4s", "c4ref", "c5"])
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="capture the timed steps in a CUDA graph (auto: steps "
                         "moving < 1 GiB, which are launch-bound from Python)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 26)
    ap.add_argument("--cpu-repeats", type=int, default=3)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    env_world = os.environ.get("WORLD_SIZE")
    if args.gpus is None:
        args.gpus = int(env_world or "1")
    if env_world is None and args.gpus > 1:
        # not under torchrun: launch one rank per GPU ourselves (same contract)
        if args.impl == "ours":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                sys.exit(f"bench.py --gpus {args.gpus}: needs {args.gpus} GPUs, "
                         f"{have} visible")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(env_world or "1")
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank "
                 f"per GPU (torchrun --nproc-per-node {args.gpus}) or drop --gpus")
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # communicator evidence in the log (NCCL's INIT lines: nranks, NVLS, ...)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    runner = {"c4": run_gemm, "c4raw": run_gemm, "c4s": run_gemm, "c4ref": run_matmul_q,
              "c5": run_sweep}.get(args.config, run_ours)
    out = runner(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
