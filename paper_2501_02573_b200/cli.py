"""Command-line front end for the device methods (reference cli.py:1-308, the file path only).

    python -m paper_2501_02573_b200.cli decode --b B.ldt --c C.ldt --v V.ldt --gamma 0.97 --decay
    python -m paper_2501_02573_b200.cli gen --seqlen 4096 --dtype bf16
    python -m paper_2501_02573_b200.cli explain --seqlen 8192 --dtype bf16
    python -m paper_2501_02573_b200.cli bench --seqlen 1024,8192 --rank 128 --dim 128 --mask decay

Same subcommand names, flags and exit codes as the reference (0 ok, 2 usage, 3 resource;
cli.py:292-304).  ``decode`` accepts per-head gammas (``--gamma 0.9,0.99``; the reference took
a scalar, cli.py:260) and LDT1 files in f32/f64/bf16 (tensorio.py; bf16 is the new dtype byte).
Host tensors go through ``run_method``'s overlapped host<->device pipeline; there is no CPU
path, so every subcommand except ``gen``/``explain`` needs the CUDA library and a GPU.
The reference's ``verify`` and ``complexity`` subcommands belong to the CPU oracle and the
opcount fitter, which are test infrastructure here (tests/, oracle/), not product code.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

from . import bench as bench_mod
from . import dispatch, tensorio
from .errors import LinAttnError, ResourceError, UsageError
from .kernels import CONCRETE_METHODS, BlockParams, MethodId, run_method
from .tensor import make_inputs


def _int_list(text: str):
    try:
        return [int(tok) for tok in text.split(",") if tok.strip()]
    except ValueError:
        raise UsageError(f"expected a comma-separated integer list, got {text!r}")


def _float_list(text: str):
    try:
        return [float(tok) for tok in text.split(",") if tok.strip()]
    except ValueError:
        raise UsageError(f"expected a comma-separated float list, got {text!r}")


def _methods(text: str):
    if text == "all":
        return list(CONCRETE_METHODS)
    return [MethodId.parse(tok.strip()) for tok in text.split(",") if tok.strip()]


def _policy(args):
    path = getattr(args, "policy", None) or os.environ.get(dispatch.POLICY_ENV_VAR)
    return dispatch.load_policy(path) if path else dispatch.default_policy()


def _host(x):
    """LDT1 payload -> torch host tensor (pinned when a GPU is present, for async H2D)."""
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    return t.pin_memory() if torch.cuda.is_available() else t


def cmd_decode(args) -> int:
    b = tensorio.read_tensor(args.b)
    c = tensorio.read_tensor(args.c)
    v = tensorio.read_tensor(args.v)
    gam = _float_list(args.gamma)
    inputs = make_inputs(_host(b), _host(c), _host(v), gamma=gam[0] if len(gam) == 1 else gam,
                         decay=args.decay)
    method = MethodId.parse(args.method)
    if method is MethodId.AUTO:
        method, _ = dispatch.explain(inputs, _policy(args))
        print(f"resolved: {method.value}", file=sys.stderr)
    out, _ = run_method(method, inputs, BlockParams(seq_parts=args.seq_parts))
    tensorio.write_tensor(out, args.out)
    print(f"wrote {args.out}")
    return 0


def cmd_gen(args) -> int:
    dtype = np.float64 if args.dtype == "f64" else np.float32
    inp = bench_mod.gen_inputs(args.batch, args.heads, args.seqlen, args.rank, args.dim, dtype, args.seed)
    for arr, path in ((inp.b, args.out_b), (inp.c, args.out_c), (inp.v, args.out_v)):
        tensorio.write_tensor(torch.from_numpy(arr).to(torch.bfloat16) if args.dtype == "bf16" else arr, path)
    print(f"wrote {args.out_b}, {args.out_c}, {args.out_v}")
    return 0


def cmd_explain(args) -> int:
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    z = torch.zeros((args.batch, args.heads, args.seqlen, 1), dtype=dt)
    inputs = make_inputs(z, z, z, decay=args.mask == "decay")
    method, rule = dispatch.explain(inputs, _policy(args))
    print(f"{method.value}  ({rule})")
    return 0


def cmd_bench(args) -> int:
    ranks, dims = _int_list(args.rank), _int_list(args.dim)
    if len(ranks) == 1:
        ranks = ranks * len(dims)
    if len(dims) == 1:
        dims = dims * len(ranks)
    if len(ranks) != len(dims):
        raise UsageError("--rank and --dim lists must pair up (equal length or length 1)")
    grid = [(bt, args.heads, n, r, d) for bt in _int_list(args.batch) for n in _int_list(args.seqlen)
            for r, d in zip(ranks, dims)]
    cfg = bench_mod.BenchConfig(methods=_methods(args.methods), grid=grid, decay=args.mask == "decay",
                                gamma=args.gamma, repeats=args.repeats, warmup=args.warmup,
                                drop_extremes=args.drop_extremes, seed=args.seed)
    text = bench_mod.render_report(bench_mod.run_bench(cfg), args.format)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)
        print(f"wrote {args.out}")
    else:
        sys.stdout.write(text)
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="linattn-b200",
                                description="B200 decayed causal linear attention on tensor files")
    sub = p.add_subparsers(dest="command", required=True)

    q = sub.add_parser("decode", help="run attention on LDT1 tensor files")
    q.add_argument("--b", required=True)
    q.add_argument("--c", required=True)
    q.add_argument("--v", required=True)
    q.add_argument("--gamma", default="1.0", help="one gamma, or one per head (comma separated)")
    q.add_argument("--decay", action="store_true")
    q.add_argument("--method", default="auto")
    q.add_argument("--seq-parts", type=int, default=2, help="segments for b200-seqpar")
    q.add_argument("--out", default="O.ldt")
    q.add_argument("--policy", default=None)
    q.set_defaults(fn=cmd_decode)

    q = sub.add_parser("gen", help="write seeded standard-normal B, C, V tensor files")
    q.add_argument("--batch", type=int, default=1)
    q.add_argument("--heads", type=int, default=1)
    q.add_argument("--seqlen", type=int, required=True)
    q.add_argument("--rank", type=int, default=16)
    q.add_argument("--dim", type=int, default=16)
    q.add_argument("--dtype", choices=["f32", "f64", "bf16"], default="f32")
    q.add_argument("--seed", type=int, default=0)
    q.add_argument("--out-b", default="B.ldt")
    q.add_argument("--out-c", default="C.ldt")
    q.add_argument("--out-v", default="V.ldt")
    q.set_defaults(fn=cmd_gen)

    q = sub.add_parser("explain", help="show which method auto would pick")
    q.add_argument("--batch", type=int, default=1)
    q.add_argument("--heads", type=int, default=1)
    q.add_argument("--seqlen", type=int, required=True)
    q.add_argument("--mask", choices=["binary", "decay"], default="binary")
    q.add_argument("--dtype", choices=["bf16", "f32"], default="f32")
    q.add_argument("--policy", default=None)
    q.set_defaults(fn=cmd_explain)

    q = sub.add_parser("bench", help="time device methods over a configuration grid (CUDA events)")
    q.add_argument("--methods", default="b200-chunked,b200-chunked-f32")
    q.add_argument("--seqlen", default="1024,8192")
    q.add_argument("--batch", default="1")
    q.add_argument("--heads", type=int, default=8)
    q.add_argument("--rank", default="128")
    q.add_argument("--dim", default="128")
    q.add_argument("--mask", choices=["binary", "decay"], default="decay")
    q.add_argument("--gamma", type=float, default=0.99)
    q.add_argument("--repeats", type=int, default=15)
    q.add_argument("--warmup", type=int, default=2)
    q.add_argument("--drop-extremes", action="store_true")
    q.add_argument("--seed", type=int, default=0)
    q.add_argument("--format", choices=["csv", "markdown"], default="markdown")
    q.add_argument("--out", default=None)
    q.set_defaults(fn=cmd_bench)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except ResourceError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except (UsageError, LinAttnError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
