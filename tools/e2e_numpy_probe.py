"""Dev probe: run_method e2e on pageable numpy inputs (the reference user's call) vs pinned torch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_02573_b200 as la
B, H, N, d = int(os.environ.get("PB", 8)), 32, 8192, 128
rng = np.random.default_rng(0)
b, c, v = (rng.standard_normal((B, H, N, d), dtype=np.float32) for _ in range(3))
gam = [1 - 2 ** (-5 - 10 * h / 31) for h in range(H)]
inp = la.make_inputs(b, c, v, gamma=gam, decay=True)
for method in ("b200-chunked", "b200-chunked-f32"):
    la.run_method(la.MethodId.parse(method), inp, validate=False)
    torch.cuda.synchronize()
    t = time.perf_counter()
    out, _ = la.run_method(la.MethodId.parse(method), inp, validate=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{method} numpy f32 pageable: {dt * 1e3:.1f} ms ({B * N / dt / 1e6:.2f} M tokens/s), out {out.dtype}", flush=True)
