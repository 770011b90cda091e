"""Dev: configs[1] end to end through run_method on pinned host bf16 tensors at several
pipeline piece counts (kernels._host_pipelined)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_02573_b200 as la
from paper_2501_02573_b200 import kernels

B, H, N, d = 8, 32, 8192, 128
q, k, v = (torch.randn(B, H, N, d, dtype=torch.bfloat16).pin_memory() for _ in range(3))
o = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
inp = la.AttnInputs(b=q, c=k, v=v, gamma=[0.99] * H, decay=True)
orig = kernels._host_pipelined
for pieces in [int(x) for x in (sys.argv[1:] or ["16", "32", "64"])]:
    kernels._host_pipelined = lambda i, c, r, res, p=16, _n=pieces: orig(i, c, r, res, _n)
    la.run_method(la.MethodId.B200_CHUNKED, inp, validate=False, out=o)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(8):
        la.run_method(la.MethodId.B200_CHUNKED, inp, validate=False, out=o)
    torch.cuda.synchronize()
    print(json.dumps({"pieces": pieces, "ms": (time.perf_counter() - t0) / 8 * 1e3}), flush=True)
kernels._host_pipelined = orig
