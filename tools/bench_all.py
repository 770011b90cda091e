"""Dev timing sweep of the prefill kernels over BASELINE.json configs[1], [2], [4] (1 GPU).

    python tools/bench_all.py [--which cfg2,cfg3,cfg5] [--iters 20]

Prints one line per case: ms, tokens/s, algorithmic GB/s and fraction of HBM peak.
Not the bench contract (bench.py is); used to compare kernel variants.
"""
import argparse
import inspect
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02573_b200 import ops  # noqa: E402

CFGS = {
    "cfg2": (8, 32, 8192, 128, 128),
    "cfg3": (4, 16, 16384, 256, 512),
    "cfg5": (1, 32, 131072, 128, 128),
    "cfg2s": (2, 32, 8192, 128, 128),
    "cfg2x": (5, 32, 8192, 128, 128),      # 160 units: 1.08 waves unbalanced
    "cfg2d": (8, 32, 8192, 64, 128),
}


def timeit(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="cfg2,cfg3,cfg5")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--modes", default="prefill,state,split")
    args = ap.parse_args()
    hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "MEASURED_PEAKS.json")))["hbm_gbs"]
    for name in args.which.split(","):
        B, H, N, dk, dv = CFGS[name]
        q = torch.randn(B, H, N, dk, device="cuda", dtype=torch.bfloat16)
        k = torch.randn_like(q)
        v = torch.randn(B, H, N, dv, device="cuda", dtype=torch.bfloat16)
        out = torch.empty_like(v)
        l2 = ops.log2_gamma([1 - 2 ** (-5 - 10 * h / max(1, H - 1)) for h in range(H)], True, "cuda")
        alg = B * H * N * ops.bytes_per_token_head(dk, dv)
        modes = args.modes.split(",")
        cases = []
        if "prefill" in modes:
            kw = {"seq_split": 1} if "seq_split" in inspect.signature(ops.prefill).parameters else {}
            cases.append(("prefill", lambda: ops.prefill(q, k, v, l2, out=out, **kw), alg))
        if "split" in modes and "seq_split" in inspect.signature(ops.prefill).parameters:
            cases.append(("prefill-auto-split", lambda: ops.prefill(q, k, v, l2, out=out), alg))
        if "state" in modes:
            cases.append(("state_pass", lambda: ops.state_pass(k, v, l2), B * H * N * 2 * (dk + dv)))
        for label, fn, nbytes in cases:
            try:
                ms = timeit(fn, args.iters)
            except TypeError:
                continue
            gbs = nbytes / ms / 1e6
            print(json.dumps({"cfg": name, "case": label, "ms": round(ms, 4),
                              "tokens_per_s": B * N / ms * 1e3, "GBps": round(gbs, 1),
                              "frac_hbm": round(gbs / hbm, 3)}), flush=True)
        del q, k, v, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
