"""Dev driver for ncu: the one-launch row recurrence (b200-recurrent) at B=8,H=32,N=2048,d=128 bf16."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
q = torch.randn(8, 32, 2048, 128, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
l2 = ops.log2_gamma([0.99] * 32, True, "cuda")
for _ in range(2):
    ops.recurrent(q, k, v, l2)
torch.cuda.synchronize()
