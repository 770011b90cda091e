"""Where the front-door time goes (configs[1] bf16 device tensors): host wall per call, synced."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_02573_b200 as la  # noqa: E402
from paper_2501_02573_b200 import ops  # noqa: E402

B, H, N, d = 8, 32, 8192, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, H, N, d, device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))
gam = [1 - 2.0 ** (-5 - 10 * h / 31) for h in range(H)]
l2 = ops.log2_gamma(gam, True, "cuda")
out = torch.empty_like(v)


def timeit(name, fn, n=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
        torch.cuda.synchronize()
    print(f"{name:40s} {1e3 * (time.perf_counter() - t0) / n:.3f} ms", flush=True)


timeit("ops.prefill + sync", lambda: ops.prefill(q, k, v, l2, out=out))
inp = la.make_inputs(q, k, v, gamma=gam, decay=True)
timeit("run_method(validate=False)", lambda: la.run_method(la.MethodId.B200_CHUNKED, inp, validate=False))
timeit("log2_gamma", lambda: ops.log2_gamma(gam, True, "cuda"))
timeit("make_inputs", lambda: la.make_inputs(q, k, v, gamma=gam, decay=True))
timeit("explain", lambda: la.explain(inp))
timeit("output scan", lambda: la.tensor._device_nonfinite([("O", out)]))
timeit("decode(inp) established", lambda: la.decode(inp))
timeit("decode(make_inputs())", lambda: la.decode(la.make_inputs(q, k, v, gamma=gam, decay=True)))
import cProfile, pstats  # noqa: E401,E402
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    la.decode(la.make_inputs(q, k, v, gamma=gam, decay=True))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
