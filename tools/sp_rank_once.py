"""Dev driver for ncu: the sequence-parallel rank path at the 8-GPU configs[4] slice, 3 times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
from paper_2501_02573_b200.sp import CudaBackend
B, H, N, d = 1, 32, 16384, 128
q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
l2 = ops.log2_gamma([1 - 2 ** (-5 - 10 * h / 31) for h in range(H)], True, "cuda")
be = CudaBackend()
gathered = torch.zeros(8, B, H, d, d, device="cuda")
for _ in range(3):
    data, end = be.local_states(k, v, l2)
    si = be.prefix_combine(gathered, [N] * 8, 7, l2)
    be.prefill(q, k, v, l2, si, data)
torch.cuda.synchronize()
