"""GPU rows for the reference's measurement engine.

Mirrors the reference ``linattn.bench`` contract -- ``BenchConfig`` / ``BenchRow`` /
``BenchReport``, ``summarize`` (bench.py:62-74), ``gen_inputs`` (bench.py:77-84),
``run_bench`` (bench.py:87-125), ``render_report`` (bench.py:216-249) -- for the device
methods, with two differences that a GPU forces:

* timing is CUDA events on the launching stream around each call (inputs resident on the
  device, output preallocated by the method as in the reference), after ``warmup`` calls;
* every row also carries roofline columns: algorithmic GB/s (q, k, v read once, o written
  once -- SURVEY.md 8(d)), the fraction of the measured HBM peak, and tensor TFLOP/s at the
  reference chunk C0 = 64 (kernels.py:57, 158-159).

``ResourceError`` becomes an ``OOM`` row exactly as in the reference (bench.py:116-117);
a CUDA out-of-memory error is mapped to the same row status.
"""

from __future__ import annotations

import json
import math
import os
import platform
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .errors import ResourceError, UsageError
from .kernels import BlockParams, MethodId, run_method
from .tensor import AttnInputs, validate_inputs

GENERATOR_NOTE = ("numpy PCG64 via default_rng, seeded per config with [seed, batch, heads, seqlen, rank, dim] "
                  "(reference bench.py:77-84), cast to the method's device dtype")
C0 = 64
_PEAKS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")


@dataclass
class BenchConfig:
    methods: list
    grid: list  # (batch, heads, seqlen, rank, dim) tuples
    decay: bool = False
    gamma: float = 0.9
    dtype: type = np.float32
    repeats: int = 15
    warmup: int = 2
    drop_extremes: bool = False
    seed: int = 0
    params: BlockParams = field(default_factory=BlockParams)


@dataclass
class BenchRow:
    method: MethodId
    batch: int
    heads: int
    seqlen: int
    rank: int
    dim: int
    mask: str
    gamma: float
    dtype: str
    mean_s: float | None
    std_s: float | None
    opcount: int | None
    status: str  # "ok" or "OOM"
    gbps: float | None = None          # algorithmic bytes / mean time
    frac_hbm: float | None = None      # of MEASURED_PEAKS.json hbm_gbs
    tflops_c64: float | None = None    # reference two-level-block flops at C0 / mean time


@dataclass
class BenchReport:
    rows: list
    meta: dict


def summarize(times, drop_extremes: bool = False):
    """(mean, sample std) of the observations, optionally dropping one max and one min first.

    Std uses the n-1 denominator; 0.0 below two samples (reference bench.py:62-74).
    """
    obs = sorted(float(t) for t in times)
    if drop_extremes:
        if len(obs) < 3:
            raise UsageError("drop_extremes needs at least 3 observations")
        obs = obs[1:-1]
    mean = sum(obs) / len(obs)
    if len(obs) < 2:
        return mean, 0.0
    var = sum((t - mean) ** 2 for t in obs) / (len(obs) - 1)
    return mean, math.sqrt(var)


def gen_inputs(batch, heads, seqlen, rank, dim, dtype=np.float32, seed=0, decay=False, gamma=0.9,
               device=None, device_dtype=None) -> AttnInputs:
    """Seeded standard-normal inputs, bitwise equal to the reference's for (config, seed).

    With ``device`` set, the arrays are moved to that device (as ``device_dtype``, default the
    torch equivalent of ``dtype``) so timed calls see resident inputs.
    """
    rng = np.random.default_rng([seed, batch, heads, seqlen, rank, dim])
    b = rng.standard_normal((batch, heads, seqlen, rank)).astype(dtype)
    c = rng.standard_normal((batch, heads, seqlen, rank)).astype(dtype)
    v = rng.standard_normal((batch, heads, seqlen, dim)).astype(dtype)
    if device is not None:
        tdt = device_dtype or (torch.float64 if np.dtype(dtype) == np.float64 else torch.float32)
        b, c, v = (torch.from_numpy(x).to(device=device, dtype=tdt) for x in (b, c, v))
    return AttnInputs(b=b, c=c, v=v, gamma=[gamma] * heads, decay=decay)


def _peaks():
    try:
        with open(_PEAKS) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0   # B200_PROFILING.md fallback


_DEVICE_DTYPE = {MethodId.B200_CHUNKED: torch.bfloat16, MethodId.B200_SEQPAR: torch.bfloat16,
                 MethodId.B200_CHUNKED_F32: torch.float32, MethodId.B200_RECURRENT: torch.float32}


def run_bench(cfg: BenchConfig) -> BenchReport:
    """Time each (config, method) on the current CUDA device (reference bench.py:87-125)."""
    if not cfg.grid:
        raise UsageError("benchmark grid is empty")
    if cfg.drop_extremes and cfg.repeats < 3:
        raise UsageError("drop_extremes requires repeats >= 3")
    for m in cfg.methods:
        if not isinstance(m, MethodId) or m is MethodId.AUTO:
            raise UsageError(f"bench needs concrete methods, got {m}")
    if not torch.cuda.is_available():
        raise ResourceError("no CUDA device: the device methods have no CPU fallback")
    hbm, tc_peak = _peaks()
    mask_name = "decay" if cfg.decay else "binary"
    rows = []
    for batch, heads, seqlen, rank, dim in cfg.grid:
        host = gen_inputs(batch, heads, seqlen, rank, dim, cfg.dtype, cfg.seed, cfg.decay, cfg.gamma)
        validate_inputs(host)
        for method in cfg.methods:
            tdt = _DEVICE_DTYPE[method]
            row = BenchRow(method, batch, heads, seqlen, rank, dim, mask_name, cfg.gamma,
                           "bf16" if tdt == torch.bfloat16 else "f32", None, None, None, "ok")
            try:
                inputs = AttnInputs(b=torch.from_numpy(host.b).to("cuda", tdt),
                                    c=torch.from_numpy(host.c).to("cuda", tdt),
                                    v=torch.from_numpy(host.v).to("cuda", tdt),
                                    gamma=host.gamma, decay=host.decay)
                opcount = None
                for _ in range(cfg.warmup):
                    _, opcount = run_method(method, inputs, cfg.params, validate=False)
                times = []
                for _ in range(cfg.repeats):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    _, opcount = run_method(method, inputs, cfg.params, validate=False)
                    e1.record()
                    e1.synchronize()
                    times.append(e0.elapsed_time(e1) * 1e-3)
                row.mean_s, row.std_s = summarize(times, cfg.drop_extremes)
                row.opcount = opcount
                elem = 2 if tdt == torch.bfloat16 else 4
                nbytes = batch * heads * seqlen * ops.bytes_per_token_head(rank, dim, elem)
                flops = 2 * batch * heads * seqlen * (C0 * (rank + dim) + 2 * rank * dim)
                row.gbps = nbytes / row.mean_s / 1e9
                row.frac_hbm = row.gbps / hbm
                row.tflops_c64 = flops / row.mean_s / 1e12
                del inputs
            except (ResourceError, torch.OutOfMemoryError):
                row.status = "OOM"
                torch.cuda.empty_cache()
            rows.append(row)
    meta = {
        "seed": cfg.seed,
        "dtype": "f32" if np.dtype(cfg.dtype) == np.float32 else "f64",
        "generator": GENERATOR_NOTE,
        "host": platform.node() or "unknown",
        "device": torch.cuda.get_device_name(),
        "timing": "CUDA events per call, device-resident inputs",
        "hbm_peak_gbs": hbm,
        "bf16_peak_tflops": tc_peak,
    }
    return BenchReport(rows=rows, meta=meta)


def _sci(x: float) -> str:
    return np.format_float_scientific(x, precision=2, exp_digits=1, trim="-")


def cell_text(row: BenchRow) -> str:
    if row.status == "OOM":
        return "OOM"
    return f"{_sci(row.mean_s)} ± {_sci(row.std_s)} ({100 * row.frac_hbm:.0f}% HBM)"


CSV_HEADER = ("method,batch,heads,seqlen,rank,dim,mask,gamma,dtype,mean_s,std_s,opcount,status,"
              "gbps,frac_hbm,tflops_c64")


def render_report(report: BenchReport, fmt: str = "csv") -> str:
    """CSV (the reference columns plus the roofline columns) or a markdown latency table."""
    if fmt == "csv":
        lines = [CSV_HEADER]
        for r in report.rows:
            def f(x):
                return "" if x is None else repr(x)
            ops_s = "" if r.opcount is None else str(r.opcount)
            lines.append(f"{r.method.value},{r.batch},{r.heads},{r.seqlen},{r.rank},{r.dim},{r.mask},"
                         f"{r.gamma},{r.dtype},{f(r.mean_s)},{f(r.std_s)},{ops_s},{r.status},"
                         f"{f(r.gbps)},{f(r.frac_hbm)},{f(r.tflops_c64)}")
        return "\n".join(lines) + "\n"
    if fmt == "markdown":
        seqlens = sorted(set(r.seqlen for r in report.rows))
        methods = []
        for r in report.rows:
            if r.method not in methods:
                methods.append(r.method)
        by_key = {}
        for r in report.rows:
            by_key.setdefault((r.method, r.seqlen), r)
        lines = ["| method | " + " | ".join(str(n) for n in seqlens) + " |",
                 "|" + "---|" * (len(seqlens) + 1)]
        for m in methods:
            cells = [cell_text(by_key[(m, n)]) if (m, n) in by_key else "" for n in seqlens]
            lines.append(f"| {m.value} | " + " | ".join(cells) + " |")
        meta = ", ".join(f"{k}: {v}" for k, v in report.meta.items())
        lines += ["", f"<!-- {meta} -->"]
        return "\n".join(lines) + "\n"
    raise UsageError(f"unknown report format {fmt!r} (expected csv or markdown)")
