"""Minimal driver for ncu: one prefill shape launched 3 times.

PROF_SHAPE="B,H,N,dk[,dv]" (default configs[1] 8,32,8192,128); PROF_SPLIT=1 forces one pass;
PROF_DTYPE=f32|bf16 (default bf16); PROF_KERNEL=auto|tc|tf32|simt.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
shape = [int(x) for x in os.environ.get("PROF_SHAPE", "8,32,8192,128").split(",")]
B, H, N, dk = shape[:4]
dv = shape[4] if len(shape) > 4 else dk
dt = torch.float32 if os.environ.get("PROF_DTYPE") == "f32" else torch.bfloat16
kern = os.environ.get("PROF_KERNEL", "auto")
q = torch.randn(B, H, N, dk, device="cuda", dtype=dt)
k = torch.randn_like(q)
v = torch.randn(B, H, N, dv, device="cuda", dtype=dt)
l2 = ops.log2_gamma([1 - 2 ** (-5 - 10 * h / max(1, H - 1)) for h in range(H)], True, "cuda")
split = 1 if os.environ.get("PROF_SPLIT") == "1" else None
for _ in range(3):
    ops.prefill(q, k, v, l2, seq_split=split, kernel=kern)
torch.cuda.synchronize()
