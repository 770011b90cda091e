"""Time the 3xTF32 prefill at the configs[1] shape (fp32), CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_02573_b200 import ops  # noqa: E402

B, H, N, d = [int(x) for x in os.environ.get("SHAPE", "8,32,8192,128").split(",")]
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, H, N, d, device="cuda", generator=g) for _ in range(3))
l2 = ops.log2_gamma([1 - 2.0 ** (-5 - 10 * h / max(1, H - 1)) for h in range(H)], True, "cuda")
out = torch.empty_like(v)
kern = os.environ.get("KERN", "tf32")
for _ in range(3):
    ops.prefill(q, k, v, l2, out=out, kernel=kern)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    ops.prefill(q, k, v, l2, out=out, kernel=kern)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"{kern} {B}x{H}x{N}x{d} balance={os.environ.get('LINATTN_BALANCE', 'auto')}: {ms:.3f} ms, "
      f"{B * H * N * 16 * d / ms / 1e6:.0f} GB/s", flush=True)
