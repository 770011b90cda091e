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
(the reference's CPU route from baseline/_ref over the whole batch, rank 0 only), ``decode`` (configs[3] decode step), ``clocks`` (nvidia-smi during
the timed region), ``gpu_launches`` (our kernels launched in the timed region).
``--impl reference`` times the reference's own CPU route (linattn.run_method from
baseline/_ref, the unmodified package; the oracle port only if it is absent) on rank 0.
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
#
# The reference's own CPU implementation of the path: ``linattn.run_method(TWO_LEVEL_BLOCK)``
# (kernels.py:139-166; the LA analogue) from the unmodified package installed into
# baseline/_ref (``__graft_entry__.build()``; pip --target), timed by the reference's protocol
# (bench.py:87-125): inputs generated BEFORE the timer, warm-up runs, then repeats of
# ``run_method(..., validate=False)`` under perf_counter, summarised by the reference's own
# ``summarize`` (mean, n-1 std).  Two figures:
#   * "pool": the configs[1] batch's (b, h) slices spread over one worker process per host core
#     with one BLAS thread each (slices are independent) -- all the host threads;
#   * "as_shipped": one process, BLAS at its default thread count, ``run_bench`` itself on a
#     sample of the batch (the reference runs strictly sequentially).
# Without baseline/_ref the numpy restatement in oracle/ stands in (kind "port").

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
REF_METHOD = "two-level-block"


def _import_reference():
    """The reference package from baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "linattn")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import linattn
    except Exception:  # a broken install: fall back to the port, and say so in the line
        return None
    return linattn


def _slice_inputs(sid, n, dk, dv, gamma):
    """Inputs of (b, h) slice `sid`: standard normal f32 like reference gen_inputs (bench.py:77-84),
    seeded per slice so every worker builds only its own slices."""
    rng = np.random.default_rng([0, sid, n, dk, dv])
    b = rng.standard_normal((1, 1, n, dk)).astype(np.float32)
    c = rng.standard_normal((1, 1, n, dk)).astype(np.float32)
    v = rng.standard_normal((1, 1, n, dv)).astype(np.float32)
    return b, c, v, gamma


def _ref_worker(conn, sids, n, dk, dv, gammas, use_ref, method_name=REF_METHOD):
    """Pool worker: builds its slices' inputs (untimed), then times run_method per command."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    lib = _import_reference() if use_ref else None
    if lib is not None:
        method = lib.MethodId.parse(method_name)
        params = lib.BlockParams()
        inputs = []
        for sid in sids:
            b, c, v, g = _slice_inputs(sid, n, dk, dv, gammas[sid % len(gammas)])
            inputs.append(lib.AttnInputs(b=b, c=c, v=v, gamma=[g], decay=True))
            lib.validate_inputs(inputs[-1])
        run = lambda inp: lib.run_method(method, inp, params, validate=False)   # noqa: E731
    else:
        from oracle import linattn_oracle as orc
        inputs = [_slice_inputs(sid, n, dk, dv, gammas[sid % len(gammas)]) for sid in sids]
        if method_name == "row-based":
            run = lambda inp: orc.row_recurrence(inp[0][0, 0], inp[1][0, 0], inp[2][0, 0], inp[3], True,  # noqa: E731
                                                 dtype=np.float32)
        else:
            run = lambda inp: orc.blocked_attn(inp[0], inp[1], inp[2], [inp[3]], True, block=C0)   # noqa: E731
    conn.send("ready")
    while True:
        cmd = conn.recv()
        if cmd is None:
            break
        times = []
        for inp in inputs:
            t0 = time.perf_counter()
            run(inp)
            times.append(time.perf_counter() - t0)
        conn.send(times)
    conn.close()


class RefPool:
    """One worker process per core, each owning a fixed share of the (b, h) slices."""

    def __init__(self, slices, workers, n, dk, dv, gammas, use_ref, method_name=REF_METHOD):
        ctx = mproc.get_context("spawn")
        self.conns, self.procs = [], []
        os.environ["OPENBLAS_NUM_THREADS"] = "1"          # inherited by the spawned workers
        for w in range(workers):
            mine = list(range(w, slices, workers))
            if not mine:
                continue
            a, b = ctx.Pipe()
            p = ctx.Process(target=_ref_worker, args=(b, mine, n, dk, dv, gammas, use_ref, method_name),
                            daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for c in self.conns:
            assert c.recv() == "ready"
        self.slices = slices

    def step(self):
        """Wall time of one pass over every slice (all workers concurrently) + per-slice times."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send("run")
        per = [t for c in self.conns for t in c.recv()]
        return time.perf_counter() - t0, per

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=30)


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), model)
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": i.get("internal_api"), "version": i.get("version"), "threads": i.get("num_threads")}
                for i in threadpool_info() if i.get("user_api") == "blas"]
    except Exception:
        pass
    return {"cpu_model": model, "cores": cores_available(), "blas": blas, "numpy": np.__version__}


def as_shipped(lib, heads=8, repeats=3):
    """The reference's run_bench (one process, default BLAS threads) on a 1 x heads x 8192 x 128
    sample of configs[1], both blocking routes; per-slice seconds (mean, std)."""
    cfg = lib.BenchConfig(methods=[lib.MethodId.TWO_LEVEL_BLOCK, lib.MethodId.BLOCK_BASED],
                          grid=[(1, heads, CFG["N"], CFG["dk"], CFG["dv"])], decay=True,
                          gamma=gammas(CFG["H"])[CFG["H"] // 2], dtype=np.float32, repeats=repeats, warmup=1)
    rep = lib.run_bench(cfg)
    return {r.method.value: {"per_slice_ms": 1e3 * r.mean_s / heads, "std_ms": 1e3 * r.std_s / heads,
                             "tokens_per_s": CFG["B"] * CFG["N"] / (r.mean_s / heads * CFG["B"] * CFG["H"])}
            for r in rep.rows if r.status == "ok"}


def cpu_arm(steps, warmup, seconds=None):
    """Time the reference CPU route on configs[1]: `steps` timed passes over the whole batch
    (or, with `seconds`, as many passes as fit, at least one).  Returns a dict for the line."""
    lib = _import_reference()
    kind = "reference" if lib is not None else "port"
    cores = cores_available()
    slices = CFG["B"] * CFG["H"]
    pool = RefPool(slices, cores, CFG["N"], CFG["dk"], CFG["dv"], gammas(CFG["H"]), lib is not None)
    try:
        for _ in range(warmup):
            pool.step()
        walls, per = [], []
        while True:
            wall, p = pool.step()
            walls.append(wall)
            per.extend(p)
            if seconds is None and len(walls) >= steps:
                break
            if seconds is not None and sum(walls) >= seconds:
                break
    finally:
        pool.close()
    if lib is not None:
        mean, std = lib.summarize(walls)
    else:
        mean, std = float(np.mean(walls)), float(np.std(walls, ddof=1)) if len(walls) > 1 else 0.0
    tokens = CFG["B"] * CFG["N"]              # one pass = the whole configs[1] batch
    out = {"value": tokens / mean, "unit": "tokens/s", "cores": cores, "kind": kind,
           "ms_per_step": 1e3 * mean, "std_ms": 1e3 * std, "passes": len(walls),
           "per_slice_ms": 1e3 * float(np.mean(per)),
           "sample": (f"the whole configs[1] batch (B=8,H=32,N=8192,d=128 f32, {slices} (b,h) slices) per pass, "
                      f"{len(walls)} timed passes after {warmup} warm-up; "
                      + (f"linattn.run_method({REF_METHOD}, validate=False) from baseline/_ref"
                         if lib is not None else "oracle port of two-level-block (baseline/_ref absent)")
                      + f", inputs generated before the timer, {len(pool.conns)} worker processes x 1 BLAS thread"),
           "host": host_info()}
    if lib is not None:
        try:
            out["as_shipped"] = as_shipped(lib)
        except Exception as exc:  # informational only
            out["as_shipped"] = {"error": repr(exc)}
    return out


def cpu_decode_arm(sample=64):
    """The reference's row recurrence (run_method(row-based), kernels.py:93-106: the per-token
    decode update S <- gamma S + k^T v, o = q S) on `sample` of the 8192 configs[3] states for
    1024 tokens each, over one worker process per core; extrapolated linearly to one decode step
    of all 8192 states (the states are independent, kernels.py:273-280)."""
    lib = _import_reference()
    cores = cores_available()
    states = DEC["B"] * DEC["H"]
    pool = RefPool(sample, cores, DEC["steps"], DEC["dk"], DEC["dv"], gammas(DEC["H"]), lib is not None,
                   method_name="row-based")
    try:
        pool.step()                                           # warm-up
        wall, per = pool.step()
    finally:
        pool.close()
    us = wall / DEC["steps"] * (states / sample) * 1e6
    return {"us_per_step": us, "cores": len(pool.conns), "kind": "reference" if lib is not None else "port",
            "per_state_token_us": 1e6 * float(np.mean(per)) / DEC["steps"],
            "sample": (f"{sample} of {states} (b,h) states x {DEC['steps']} tokens, d={DEC['dk']} f32, "
                       + ("linattn.run_method(row-based, validate=False) from baseline/_ref"
                          if lib is not None else "oracle port of the row recurrence")
                       + f", {len(pool.conns)} worker processes x 1 BLAS thread; one decode step of all "
                         f"{states} states extrapolated linearly")}


def cores_available():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    arm = cpu_arm(args.steps, args.warmup)
    value = arm["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": arm["passes"], "warmup": args.warmup,
        "ms_per_step": arm["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (standard normal, seeded per slice)",
        "config": {"workload": "configs[1] chunked prefill B=8,H=32,N=8192,d=128 (the reference CPU route, f32)",
                   "global_batch": CFG["B"], "seq_len": CFG["N"], "heads": CFG["H"],
                   "parallelism": f"cpu process pool x{arm['cores']}", "method": REF_METHOD},
        "cpu_baseline": arm,
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
        # sampling interval: the guide's nvidia-smi recipe samples every 200 ms; every 10 ms still
        # gives several samples inside the shortest timed region without NVML traffic at 2 ms
        self.interval_s = float(os.environ.get("LINATTN_CLOCK_MS", "10")) / 1e3
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
            self._stop.wait(self.interval_s)

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
                "reasons": reasons, "samples": len(sm),
                "source": f"nvml, every {self.interval_s * 1e3:g} ms, inside the timed region"}


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


def bench_cfg3(args, ops, dev, g, hbm, tc_burst, tc_sus, barrier, max_over_ranks):
    """configs[2]: B=4, H=16, N=16384, dk=256, dv=512 bf16 (per GPU; weak scaling over ranks).

    Tensor-heavy and timed back to back, so the board's power cap pulls the SM clock below max
    (the clocks seen are reported): the fraction is given against the burst AND the sustained
    (power-capped) bf16 peak of MEASURED_PEAKS.json (the recipe's denominator for a kernel timed
    inside a long loop)."""
    import torch
    B, H, N, dk, dv = 4, 16, 16384, 256, 512
    q = torch.randn(B, H, N, dk, device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn(B, H, N, dk, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(B, H, N, dv, device=dev, dtype=torch.bfloat16, generator=g)
    out = torch.empty_like(v)
    l2 = ops.log2_gamma(gammas(H), True, dev)
    with ClockSampler(torch.cuda.current_device()) as clk:
        clk.mark("start")
        ms = _time_events(lambda: ops.prefill(q, k, v, l2, out=out), 20, barrier, max_over_ranks)
        clk.mark("end")
    nbytes = B * H * N * ops.bytes_per_token_head(dk, dv)
    flops = 2 * B * H * N * (C0 * (dk + dv) + 2 * dk * dv)
    gbs = nbytes / (ms * 1e-3) / 1e9
    tf = flops / (ms * 1e-3) / 1e12
    del q, k, v, out
    return {"workload": "configs[2] B=4,H=16,N=16384,dk=256,dv=512 bf16 chunked prefill per GPU",
            "ms_per_step": ms, "tokens_per_s": B * N / (ms * 1e-3), "hbm_gbs": gbs, "frac_of_hbm": gbs / hbm,
            "tensor_tflops_c64": tf, "tensor_frac_of_burst": tf / tc_burst,
            "tensor_frac_of_sustained": tf / tc_sus if tc_sus else None, "bytes_per_step": nbytes,
            "clocks": clk.summary(),
            "tensor_tflops_executed": executed_mma_flops(B, H, N, dk, dv) / (ms * 1e-3) / 1e12,
            "tensor_frac_executed_of_burst": executed_mma_flops(B, H, N, dk, dv) / (ms * 1e-3) / 1e12 / tc_burst,
            "kernel": "prefill_tc (dk=256: state in TMEM)"}


def bench_fp32(args, ops, dev, g, hbm, tc_burst, barrier, max_over_ranks):
    """configs[1] shape in fp32 -- the reference's own arithmetic type: the fp32 parity mode
    (<= 1e-4 vs the f64 oracle), 3xTF32 on the tensor cores (the default route for fp32 inputs),
    with the FFMA kernel it replaced timed beside it."""
    import torch
    B, H, N, d = 8, 32, 8192, 128
    q = torch.randn(B, H, N, d, device=dev, dtype=torch.float32, generator=g)
    k = torch.randn(B, H, N, d, device=dev, dtype=torch.float32, generator=g)
    v = torch.randn(B, H, N, d, device=dev, dtype=torch.float32, generator=g)
    out = torch.empty_like(v)
    l2 = ops.log2_gamma(gammas(H), True, dev)
    ms = _time_events(lambda: ops.prefill(q, k, v, l2, out=out, kernel="auto"), 10, barrier, max_over_ranks)
    ms_simt = _time_events(lambda: ops.prefill(q, k, v, l2, out=out, kernel="simt"), 3, barrier, max_over_ranks)
    nbytes = B * H * N * 4 * 4 * d
    # tcgen05 kind::tf32 flops issued per 32-token chunk and 128-wide dv tile, 3 products each:
    # MMA1 at M = 64 (K = dk), dS^T (N = dk, K = 32), O_intra (N = 32, K = 32), O_inter (N = 32, K = dk)
    per_chunk = 3 * 2 * (64 * 32 * d + 128 * d * 32 + 128 * 32 * 32 + 128 * 32 * d)
    tf_exec = B * H * (N // 32) * per_chunk / (ms * 1e-3) / 1e12
    tf32_peak = tc_burst / 2        # kind::tf32 issues K = 8 per MMA at the kind::f16 rate (K = 16)
    del q, k, v, out
    return {"workload": "configs[1] shape B=8,H=32,N=8192,d=128 in fp32 (b200-chunked-f32)",
            "ms_per_step": ms, "tokens_per_s": B * N / (ms * 1e-3),
            "hbm_gbs": nbytes / (ms * 1e-3) / 1e9, "frac_of_hbm": nbytes / (ms * 1e-3) / 1e9 / hbm,
            "bytes_per_step": nbytes,
            "tf32_tflops_executed": tf_exec, "tf32_frac_executed_of_peak": tf_exec / tf32_peak,
            "tf32_peak_tflops": tf32_peak, "tf32_peak_kind": "measured bf16 burst / 2",
            "kernel": ops.prefill_kernel_name(d, d, torch.float32) + " (3xTF32 tcgen05 kind::tf32)",
            "ffma_kernel_ms": ms_simt}


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

    # the public front door on device tensors: la.decode(la.make_inputs(q, k, v, ...)) per step
    # (shape/gamma validation, the deferred NaN/Inf check, auto dispatch, one prefill), host wall
    # clock with a device synchronisation per step, against the bare kernel's device time
    front = None
    if not args.no_extra:
        la.decode(la.make_inputs(q, k, v, gamma=gam, decay=True))
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(10):
            la.decode(la.make_inputs(q, k, v, gamma=gam, decay=True))
        torch.cuda.synchronize()
        fd_ms = max_over_ranks((time.perf_counter() - t0) / 10 * 1e3)
        front = {"api": "la.decode(la.make_inputs(q, k, v, gamma, decay=True)) on configs[1] CUDA bf16 tensors",
                 "ms_per_call": fd_ms, "bare_kernel_ms": ms, "ratio_to_bare_kernel": fd_ms / ms}

    # decode step (configs[3]): 1024 single-token steps, state 256x32x128x128 fp32 (512 MiB)
    dec = None
    if not args.no_decode:
        dec = bench_decode(args, ops, dev, g, hbm, barrier, max_over_ranks)

    # configs[2] (RetNet-shaped, dk=256, dv=512) prefill, and configs[4] long context: sequence
    # split inside the GPU at N=1, sequence parallel over the ranks (one NCCL all-gather) at N>1
    cfg3 = None if args.no_extra else bench_cfg3(args, ops, dev, g, hbm, tc_burst, tc_sus, barrier, max_over_ranks)
    cfg5 = None if args.no_extra else bench_seqpar(args, ops, dev, g, hbm, world, rank, barrier, max_over_ranks)
    f32 = None if args.no_extra else bench_fp32(args, ops, dev, g, hbm, tc_burst, barrier, max_over_ranks)

    # CPU baseline: the reference's own CPU route (baseline/_ref), rank 0 at N=1 only, ~10 s
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_arm(0, 1, seconds=args.cpu_seconds)
        if dec is not None:
            dec["cpu_baseline"] = cpu_decode_arm()

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
        "front_door": front,
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return run_ours(args)


def relaunch(n):
    """--gpus N outside torchrun: re-run this command as N ranks (one process per GPU)."""
    import socket
    import subprocess
    if os.environ.get("LINATTN_BENCH_BACKEND", "nccl") == "nccl":
        import torch
        have = torch.cuda.device_count()
        if have < n:
            raise SystemExit(f"bench.py: --gpus {n} needs {n} GPUs for NCCL, this host has {have} "
                             "(LINATTN_BENCH_BACKEND=gloo runs the ranks on shared GPUs as a path check)")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
