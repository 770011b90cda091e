"""Minimal driver for ncu: configs[1] prefill launched 3 times (bf16, B=8,H=32,N=8192,d=128)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
B, H, N, d = [int(x) for x in os.environ.get("PROF_SHAPE", "8,32,8192,128").split(",")]
q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
l2 = ops.log2_gamma([1 - 2 ** (-5 - 10 * h / (H - 1)) for h in range(H)], True, "cuda")
for _ in range(3):
    ops.prefill(q, k, v, l2)
torch.cuda.synchronize()
