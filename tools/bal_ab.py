"""Same-process A/B of plain vs balanced launches (LINATTN_BALANCE is read once per process, so
each configuration runs in its own process): prints ms per launch."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_02573_b200 import ops  # noqa: E402

B, H, N, dk, dv = [int(x) for x in os.environ["SHAPE"].split(",")]
dt = torch.float32 if os.environ.get("DT") == "f32" else torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(B, H, N, dk, device="cuda", generator=g).to(dt)
k = torch.randn(B, H, N, dk, device="cuda", generator=g).to(dt)
v = torch.randn(B, H, N, dv, device="cuda", generator=g).to(dt)
l2 = ops.log2_gamma([1 - 2.0 ** (-5 - 10 * h / max(1, H - 1)) for h in range(H)], True, "cuda")
out = torch.empty_like(v)
for _ in range(3):
    ops.prefill(q, k, v, l2, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ops.prefill(q, k, v, l2, out=out)
e1.record()
torch.cuda.synchronize()
print(f"{os.environ['SHAPE']} {dt} balance={os.environ.get('LINATTN_BALANCE', 'auto')}: "
      f"{e0.elapsed_time(e1) / 20:.3f} ms", flush=True)
