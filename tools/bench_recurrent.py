"""Dev timing of the one-launch row recurrence (b200-recurrent) at configs[1] size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
for dt in (torch.bfloat16, torch.float32):
    q = torch.randn(8, 32, 8192, 128, device="cuda", dtype=dt)
    k, v = torch.randn_like(q), torch.randn_like(q)
    l2 = ops.log2_gamma([0.99] * 32, True, "cuda")
    f = lambda: ops.recurrent(q, k, v, l2)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); f(); f(); e1.record(); torch.cuda.synchronize()
    print(dt, round(e0.elapsed_time(e1) / 2, 3), "ms")
