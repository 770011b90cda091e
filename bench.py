"""Benchmark: chunked prefill tokens/s on configs[1] (B=8, H=32, N=8192, d=128, bf16).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one pass of the hot path over one batch: a single chunked-prefill
launch over [B, H, N, d] bf16 Q/K/V already resident in HBM (``value``), and
the same call through the public API with pinned HOST buffers, H2D + D2H inside
the timed region (``e2e``).  Multi-GPU: one process per GPU (torchrun), batch x
head sharding with no data-path collective -> each rank runs the full configs[1]
batch ("scaling": "weak"); the timed region is bracketed by barrier +
synchronize and the max over ranks is reported.

Extra keys: ``roofline`` (dominant kernel vs MEASURED_PEAKS.json), ``cpu_baseline``
(the oracle port of the reference's CPU blocking route on a bounded sample,
rank 0 only), ``decode`` (configs[3] decode step), ``clocks`` (nvidia-smi during
the timed region), ``gpu_launches`` (our kernels launched in the timed region).
``--impl reference`` times the reference's CPU algorithm (oracle port; the
reference is pure Python/numpy and cannot travel to the GPU box) on rank 0.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mproc
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefill tokens/s @N=8K,d=128 bf16 (% TC peak); decode-step us & HBM GB/s"
CFG = dict(B=8, H=32, N=8192, dk=128, dv=128)           # BASELINE.json configs[1]
DEC = dict(B=256, H=32, dk=128, dv=128, steps=1024)     # BASELINE.json configs[3]
C0 = 64                                                  # reference default chunk (kernels.py:57)


def gammas(h):
    """Per-head gamma_h = 1 - 2^(-5 - 10 h / (H-1))."""
    return [1.0 - 2.0 ** (-5 - 10 * i / max(1, h - 1)) for i in range(h)]


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", 0)), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, 1400.0, "fallback"


# --------------------------------------------------------------------------- CPU arm

def _cpu_slice(args):
    """One (b, h) slice of the reference CPU blocking route, f32 (oracle port)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import linattn_oracle as orc
    n, dk, dv, gamma, seed = args
    rng = np.random.default_rng(seed)
    b = rng.standard_normal((1, 1, n, dk)).astype(np.float32)
    c = rng.standard_normal((1, 1, n, dk)).astype(np.float32)
    v = rng.standard_normal((1, 1, n, dv)).astype(np.float32)
    t0 = time.perf_counter()
    orc.blocked_attn(b, c, v, [gamma], True, block=C0)
    return time.perf_counter() - t0


def cpu_sample(pool, cores, per_core=1, seed=0):
    """Time cores*per_core slices of configs[1] in a process pool; tokens/s equivalent."""
    g = gammas(CFG["H"])
    jobs = [(CFG["N"], CFG["dk"], CFG["dv"], g[i % CFG["H"]], seed + i) for i in range(cores * per_core)]
    t0 = time.perf_counter()
    pool.map(_cpu_slice, jobs, chunksize=1)
    dt = time.perf_counter() - t0
    slices = len(jobs)
    tokens = slices / (CFG["B"] * CFG["H"]) * CFG["B"] * CFG["N"]  # a token passes through all H heads
    return tokens / dt, dt, slices


def cores_available():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = cores_available()
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ctx = mproc.get_context("spawn")
    with ctx.Pool(cores) as pool:
        for _ in range(args.warmup):
            cpu_sample(pool, cores)
        vals, times = [], []
        for i in range(args.steps):
            v, dt, slices = cpu_sample(pool, cores, seed=1000 + i)
            vals.append(v)
            times.append(dt)
    value = float(np.mean(vals))
    sample = (f"{slices} of {CFG['B'] * CFG['H']} (b,h) slices of configs[1] per step, f32, "
              f"two-level-block chunk {C0}, process pool x{cores}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "configs[1] chunked prefill B=8,H=32,N=8192,d=128 (bounded CPU sample)",
                   "global_batch": CFG["B"], "seq_len": CFG["N"], "parallelism": "cpu-process-pool"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm

class ClockSampler:
    """SM clock and throttle reasons sampled (NVML, every 5 ms) during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = None

    def _run(self):
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self._stop.is_set():
            mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            mem = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
            mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            try:
                watts = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
            except pynvml.NVMLError:
                watts = None
            self.samples.append((time.perf_counter(), mhz, mask, mem, watts))
            self._ready.set()
            self._stop.wait(0.002)

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
        except Exception:  # no NVML: report no samples rather than fail the bench
            return self
        self._stop = threading.Event()
        self._ready = threading.Event()
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        self._ready.wait(2.0)
        return self

    def mark(self, which):
        setattr(self, "t_" + which, time.perf_counter())

    def __exit__(self, *exc):
        if self._stop is not None:
            self._stop.set()
            self._thread.join()

    def summary(self):
        t0, t1 = getattr(self, "t_start", None), getattr(self, "t_end", None)
        inside = [s for s in self.samples if t0 is not None and t0 <= s[0] <= t1] or self.samples
        sm = [s[1] for s in inside]
        mem = [s[3] for s in inside]
        watts = [s[4] for s in inside if s[4] is not None]
        reasons = sorted({n for s in inside for n, bit in self.REASONS.items() if s[2] & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "mem_mhz": statistics.median(mem) if mem else None,
                "power_w_max": max(watts) if watts else None,
                "reasons": reasons, "samples": len(sm), "source": "nvml, 2 ms, inside the timed region"}


def load_profile_traffic(kernel_key):
    """dram bytes per launch of the dominant kernel from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(kernel_key, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def executed_mma_flops(B, H, N, dk, dv):
    """Tensor-core flops the prefill kernels actually issue, per launch.

    Per 64-token chunk and 128-wide dv tile: MMA1 P^T = K Q^T at M = 128 (64 live rows),
    dS / S update = V^T K' (N = dk), O_intra = V^T P^T (K = 64), O_inter = S^T Q^T (K = dk).
    Differs from the algorithmic count (reference chunk C0 = 64) by the M padding of MMA1 and
    by MMA1 being repeated for every dv tile.  Reported labelled as executed, not algorithmic.
    """
    chunks = -(-N // C0)
    tiles = -(-dv // 128)
    per_chunk_tile = 2 * 128 * 64 * dk + 2 * 128 * dk * 64 + 2 * 128 * 64 * 64 + 2 * 128 * 64 * dk
    return B * H * tiles * chunks * per_chunk_tile


def _time_events(fn, iters, barrier, max_over_ranks):
    """Mean ms per call over `iters` calls, CUDA events on the current stream, max over ranks."""
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return max_over_ranks(e0.elapsed_time(e1) / iters)


def bench_decode(args, ops, dev, g, hbm, barrier, max_over_ranks):
    import torch
    DB, DH, ddk, ddv = DEC["B"], DEC["H"], DEC["dk"], DEC["dv"]
    T = max(64, args.decode_steps // 64 * 64)
    state = torch.zeros(DB, DH, ddk, ddv, device=dev, dtype=torch.float32)
    qd = torch.randn(DB, DH, ddk, device=dev, dtype=torch.bfloat16, generator=g) * 0.1
    kd = torch.randn(DB, DH, ddk, device=dev, dtype=torch.bfloat16, generator=g) * 0.1
    vd = torch.randn(DB, DH, ddv, device=dev, dtype=torch.bfloat16, generator=g) * 0.1
    od = torch.empty_like(vd)
    l2d = ops.log2_gamma(gammas(DH), True, dev)
    for _ in range(3):
        ops.decode_step(qd, kd, vd, state, l2d, out=od)
    torch.cuda.synchronize()
    per_graph = 64
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            for _ in range(per_graph):
                ops.decode_step(qd, kd, vd, state, l2d, out=od)
    torch.cuda.current_stream().wait_stream(s)
    graph.replay()
    torch.cuda.synchronize()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    d0.record()
    for _ in range(T // per_graph):
        graph.replay()
    d1.record()
    torch.cuda.synchronize()
    us = max_over_ranks(d0.elapsed_time(d1) * 1e3 / T)
    dbytes = DB * DH * (2 * 4 * ddk * ddv + 2 * (2 * ddk + 2 * ddv))
    gbs = dbytes / (us * 1e-6) / 1e9
    return {"workload": f"configs[3] decode step B=256,H=32,d=128, fp32 state, bf16 q/k/v/o, {T} steps "
                        "(CUDA graph of 64 steps)",
            "us_per_step": us, "hbm_gbs": gbs, "frac_of_hbm": gbs / hbm,
            "bytes_per_step": dbytes, "steps": T, "kernel": "decode_step"}


def bench_cfg3(args, ops, dev, g, hbm, tc_burst, barrier, max_over_ranks):
    """configs[2]: B=4, H=16, N=16384, dk=256, dv=512 bf16 (per GPU; weak scaling over ranks)."""
    import torch
    B, H, N, dk, dv = 4, 16, 16384, 256, 512
    q = torch.randn(B, H, N, dk, device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn(B, H, N, dk, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(B, H, N, dv, device=dev, dtype=torch.bfloat16, generator=g)
    out = torch.empty_like(v)
    l2 = ops.log2_gamma(gammas(H), True, dev)
    ms = _time_events(lambda: ops.prefill(q, k, v, l2, out=out), 20, barrier, max_over_ranks)
    nbytes = B * H * N * ops.bytes_per_token_head(dk, dv)
    flops = 2 * B * H * N * (C0 * (dk + dv) + 2 * dk * dv)
    gbs = nbytes / (ms * 1e-3) / 1e9
    tf = flops / (ms * 1e-3) / 1e12
    del q, k, v, out
    return {"workload": "configs[2] B=4,H=16,N=16384,dk=256,dv=512 bf16 chunked prefill per GPU",
            "ms_per_step": ms, "tokens_per_s": B * N / (ms * 1e-3), "hbm_gbs": gbs, "frac_of_hbm": gbs / hbm,
            "tensor_tflops_c64": tf, "tensor_frac_of_burst": tf / tc_burst, "bytes_per_step": nbytes,
            "tensor_tflops_executed": executed_mma_flops(B, H, N, dk, dv) / (ms * 1e-3) / 1e12,
            "tensor_frac_executed_of_burst": executed_mma_flops(B, H, N, dk, dv) / (ms * 1e-3) / 1e12 / tc_burst,
            "kernel": "prefill_tc (dk=256: state in TMEM)"}


def bench_fp32(args, ops, dev, g, hbm, barrier, max_over_ranks):
    """configs[1] shape in fp32 -- the reference's own arithmetic type: the fp32 parity mode
    (FFMA kernel, <= 1e-4 vs the f64 oracle), the default route for fp32 inputs."""
    import torch
    B, H, N, d = 8, 32, 8192, 128
    q = torch.randn(B, H, N, d, device=dev, dtype=torch.float32, generator=g)
    k = torch.randn(B, H, N, d, device=dev, dtype=torch.float32, generator=g)
    v = torch.randn(B, H, N, d, device=dev, dtype=torch.float32, generator=g)
    out = torch.empty_like(v)
    l2 = ops.log2_gamma(gammas(H), True, dev)
    ms = _time_events(lambda: ops.prefill(q, k, v, l2, out=out, kernel="simt"), 5, barrier, max_over_ranks)
    # FFMA work the kernel issues per (token, head) at chunk 32 and 64-wide dv tiles (two tiles):
    # Q.K over the causal half of each chunk, A.V, Q.S, and the K^T V state update
    fma = B * H * N * (2 * (17 * d) + 2 * (17 * 64) + 2 * (d * 64) + 2 * (d * 64))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = sms * 128 * 2 * 1.965e9 / 1e12          # FP32 FFMA TFLOP/s at the 1965 MHz max clock
    tf = 2 * fma / (ms * 1e-3) / 1e12
    del q, k, v, out
    return {"workload": "configs[1] shape B=8,H=32,N=8192,d=128 in fp32 (b200-chunked-f32)",
            "ms_per_step": ms, "tokens_per_s": B * N / (ms * 1e-3),
            "hbm_gbs": B * H * N * 4 * 4 * d / (ms * 1e-3) / 1e9,
            "ffma_tflops_issued": tf, "ffma_frac_of_peak": tf / peak, "ffma_peak_tflops": peak,
            "kernel": "prefill_simt (fp32 FFMA, cp.async staging, balanced schedule)"}


def bench_seqpar(args, ops, dev, g, hbm, world, rank, barrier, max_over_ranks):
    """configs[4]: B=1, H=32, N=131072, d=128 -- one job; N>1: sequence parallel over ranks."""
    import torch
    from paper_2501_02573_b200 import sp
    B, H, N, d = 1, 32, 131072, 128
    lo, hi = sp.segment_bounds(N, world)[rank]
    lens = [b - a for a, b in sp.segment_bounds(N, world)]
    q = torch.randn(B, H, hi - lo, d, device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    l2 = ops.log2_gamma(gammas(H), True, dev)
    if world == 1:
        fn = lambda: ops.prefill(q, k, v, l2)   # noqa: E731  (sequence split inside the GPU)
        how = "sequence split inside one GPU: segment state pass -> seeded segments in parallel"
    else:
        fn = lambda: sp.sp_prefill(q, k, v, l2, lens)   # noqa: E731
        how = (f"sequence parallel over {world} GPUs: per-rank split state pass -> NCCL all_gather of "
               "[B,H,dk,dv] fp32 end states -> prefix combine -> seeded split prefill")
    ms = _time_events(fn, 20, barrier, max_over_ranks)
    nbytes = B * H * N * ops.bytes_per_token_head(d, d)
    gbs = nbytes / (ms * 1e-3) / 1e9
    plan = ops.seq_plan(B, H, hi - lo, d, d)
    del q, k, v
    return {"workload": f"configs[4] B=1,H=32,N=131072,d=128 bf16 prefill, {world} GPU(s), strong scaling",
            "ms_per_step": ms, "tokens_per_s": N / (ms * 1e-3),
            "hbm_gbs_single_pass_bytes": gbs, "frac_of_hbm_per_gpu": gbs / hbm / world,
            "method": how, "per_rank_plan": {"seg_len": plan[0], "segments": plan[1], "state_pass_split": plan[2]}}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2501_02573_b200 import _lib, ops
    import paper_2501_02573_b200 as la

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # LINATTN_BENCH_BACKEND=gloo runs the N>1 code path on a box with fewer GPUs than ranks
    # (ranks share devices; a path check, not a measurement). The default is NCCL, one GPU each.
    backend = os.environ.get("LINATTN_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:   # torchrun sets OMP_NUM_THREADS=1: give each rank its share of host cores for
        # the host-side copies of the e2e legs (pinned staging of numpy inputs)
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        torch.set_num_threads(max(1, len(os.sched_getaffinity(0)) // local_world))
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    hbm, tc_burst, tc_sus, peak_kind = peaks()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    B, H, N, dk, dv = CFG["B"], CFG["H"], CFG["N"], CFG["dk"], CFG["dv"]
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    q = torch.randn(B, H, N, dk, device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn(B, H, N, dk, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(B, H, N, dv, device=dev, dtype=torch.bfloat16, generator=g)
    gam = gammas(H)
    l2 = ops.log2_gamma(gam, True, dev)
    out = torch.empty_like(v)
    kernel = os.environ.get("LINATTN_BENCH_KERNEL", "auto")

    def step():
        ops.prefill(q, k, v, l2, out=out, kernel=kernel)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        clk.mark("start")
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark("end")
        barrier()
    launches = _lib.launch_count() - launches0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    tokens_per_rank = B * N
    value = world * tokens_per_rank / (ms * 1e-3)

    # roofline of the dominant (only) kernel in the step: algorithmic bytes / launch duration
    bytes_launch = B * H * N * ops.bytes_per_token_head(dk, dv)
    flops_launch = 2 * B * H * N * (C0 * (dk + dv) + 2 * dk * dv)
    achieved_gbs = bytes_launch / (ms * 1e-3) / 1e9
    tflops = flops_launch / (ms * 1e-3) / 1e12

    # e2e: public API with pinned host buffers, H2D + kernel + D2H in the timed region
    e2e_steps = max(3, min(args.steps, 10))
    qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
    oh = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    inputs = la.AttnInputs(b=qh, c=kh, v=vh, gamma=gam, decay=True)
    la.run_method(la.MethodId.B200_CHUNKED, inputs, validate=False, out=oh)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        la.run_method(la.MethodId.B200_CHUNKED, inputs, validate=False, out=oh)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    del qh, kh, vh, oh, inputs

    # the reference's own calling convention: pageable numpy f32 arrays (make_inputs), the method
    # auto resolves to for f32 (the fp32 parity route), validate=False as in the reference bench
    e2e_np = None
    if not args.no_extra:
        npin = [x.float().cpu().numpy() for x in (q, k, v)]
        inputs = la.make_inputs(*npin, gamma=gam, decay=True)
        meth = la.default_policy().resolve(B, N, True, "f32")[0]
        la.run_method(meth, inputs, validate=False)
        barrier()
        t0 = time.perf_counter()
        for _ in range(3):
            la.run_method(meth, inputs, validate=False)
        torch.cuda.synchronize()
        np_s = max_over_ranks((time.perf_counter() - t0) / 3)
        e2e_np = {"value": world * tokens_per_rank / np_s, "unit": "tokens/s", "ms_per_step": np_s * 1e3,
                  "h2d_bytes_per_step": 3 * B * H * N * dk * 4, "d2h_bytes_per_step": B * H * N * dv * 4,
                  "api": f"run_method({meth.value}) on pageable numpy f32 arrays (pinned staging inside)"}
        del npin, inputs

    # decode step (configs[3]): 1024 single-token steps, state 256x32x128x128 fp32 (512 MiB)
    dec = None
    if not args.no_decode:
        dec = bench_decode(args, ops, dev, g, hbm, barrier, max_over_ranks)

    # configs[2] (RetNet-shaped, dk=256, dv=512) prefill, and configs[4] long context: sequence
    # split inside the GPU at N=1, sequence parallel over the ranks (one NCCL all-gather) at N>1
    cfg3 = None if args.no_extra else bench_cfg3(args, ops, dev, g, hbm, tc_burst, barrier, max_over_ranks)
    cfg5 = None if args.no_extra else bench_seqpar(args, ops, dev, g, hbm, world, rank, barrier, max_over_ranks)
    f32 = None if args.no_extra else bench_fp32(args, ops, dev, g, hbm, barrier, max_over_ranks)

    # CPU baseline (oracle port of the reference's CPU blocking route), rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = cores_available()
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        with mproc.get_context("spawn").Pool(cores) as pool:
            cpu_sample(pool, cores)                       # warm the workers
            total_t, total_slices, rounds = 0.0, 0, 0
            while total_t < args.cpu_seconds:             # ~10 s of CPU work by default
                _, cdt, slices = cpu_sample(pool, cores, per_core=4, seed=77 + rounds)
                total_t += cdt
                total_slices += slices
                rounds += 1
        cv = total_slices / (B * H) * B * N / total_t
        cpu = {"value": cv, "unit": "tokens/s", "cores": cores, "kind": "port",
               "sample": f"{total_slices} (b,h) slices of configs[1] ({total_slices / (B * H):.1f} x the batch), "
                         f"f32 two-level-block chunk {C0} (oracle/linattn_oracle.py), process pool x{cores}, "
                         f"{total_t:.1f} s"}

    kernel_name = ops.prefill_kernel_name(dk, dv, torch.bfloat16, kernel)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (torch.randn bf16, seeded)",
        "config": {"workload": "configs[1] chunked prefill B=8,H=32,N=8192,dk=dv=128 per GPU",
                   "global_batch": B * world, "seq_len": N, "heads": H, "parallelism": f"batch x head, {world} rank(s)",
                   "gamma": "1-2^(-5-10h/(H-1))", "l2": "no flush: 1.5 GiB of inputs per step > 126 MB L2",
                   "kernel": kernel_name},
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                     "frac": achieved_gbs / hbm, "traffic": load_profile_traffic(kernel_name),
                     "peak_kind": peak_kind, "bytes_per_launch": bytes_launch,
                     "tensor_tflops_c64": tflops, "tensor_frac_of_burst": tflops / tc_burst,
                     "tensor_tflops_executed": executed_mma_flops(B, H, N, dk, dv) / (ms * 1e-3) / 1e12,
                     "tensor_frac_executed_of_burst":
                         executed_mma_flops(B, H, N, dk, dv) / (ms * 1e-3) / 1e12 / tc_burst},
        "e2e": {"value": world * tokens_per_rank / e2e_s, "unit": "tokens/s",
                "h2d_bytes_per_step": 3 * B * H * N * dk * 2, "d2h_bytes_per_step": B * H * N * dv * 2,
                "ms_per_step": e2e_s * 1e3,
                "api": "run_method(b200-chunked) on pinned host bf16 tensors (H2D | kernel | D2H overlapped per batch piece)"},
        "e2e_numpy_f32": e2e_np,
        "gpu_launches": int(max_over_ranks(launches)),
        "clocks": clk.summary(),
        "decode": dec,
        "prefill_configs2": cfg3,
        "seqpar_configs4": cfg5,
        "prefill_fp32_configs1": f32,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU-baseline sample length")
    ap.add_argument("--no-extra", action="store_true", help="skip the configs[2]/configs[4] sub-benchmarks")
    ap.add_argument("--decode-steps", type=int, default=DEC["steps"],
                    help="decode steps timed for the configs[3] sub-benchmark (multiple of 64)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
