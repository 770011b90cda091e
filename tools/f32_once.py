"""Dev driver for ncu: the fp32 FFMA prefill at B=8,H=32,N=2048,d=128, twice."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
B, H, N, d = 8, 32, 2048, 128
q = torch.randn(B, H, N, d, device="cuda"); k, v = torch.randn_like(q), torch.randn_like(q)
l2 = ops.log2_gamma([0.99] * H, True, "cuda")
for _ in range(2): ops.prefill(q, k, v, l2, kernel="simt")
torch.cuda.synchronize()
