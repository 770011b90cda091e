"""Dev probe: run_method e2e time on pinned host tensors vs the host-pipeline piece count."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_02573_b200 as la
from paper_2501_02573_b200 import kernels
B, H, N, d = 8, 32, 8192, 128
qh, kh, vh = (torch.randn(B, H, N, d, dtype=torch.bfloat16).pin_memory() for _ in range(3))
oh = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
gam = [1 - 2 ** (-5 - 10 * h / 31) for h in range(H)]
inputs = la.AttnInputs(b=qh, c=kh, v=vh, gamma=gam, decay=True)
orig = kernels._pieces
for target in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4,8,16,32,64").split(",")]:
    kernels._pieces = lambda b, h, target=target: orig(b, h, target)
    la.run_method(la.MethodId.B200_CHUNKED, inputs, validate=False, out=oh)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        la.run_method(la.MethodId.B200_CHUNKED, inputs, validate=False, out=oh)
    torch.cuda.synchronize()
    print(f"pieces~{target}: {(time.perf_counter() - t) / 5 * 1e3:.1f} ms", flush=True)
