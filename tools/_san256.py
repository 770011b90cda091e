import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
q = torch.randn(1, 40, 200, 256, device="cuda", dtype=torch.bfloat16)
k = torch.randn_like(q)
v = torch.randn(1, 40, 200, 512, device="cuda", dtype=torch.bfloat16)
ops.prefill(q, k, v, ops.log2_gamma([0.9] * 40, True, "cuda"), s_out=torch.empty(1, 40, 256, 512, device="cuda"))
torch.cuda.synchronize()
print("done")
