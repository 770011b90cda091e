"""Dev timing of the fp32 parity mode (FFMA kernel) at configs[0] and a configs[1]-sized input."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
for (B, H, N, d) in [(1, 8, 2048, 64), (8, 32, 8192, 128), (1, 32, 32768, 128)]:
    q = torch.randn(B, H, N, d, device="cuda")
    k, v = torch.randn_like(q), torch.randn_like(q)
    l2 = ops.log2_gamma([1 - 2 ** (-5 - h) for h in range(H)], True, "cuda")
    f = lambda: ops.prefill(q, k, v, l2, kernel="simt")
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"shape": [B, H, N, d], "ms": round(e0.elapsed_time(e1) / 5, 3),
                      "plan": ops.seq_plan(B, H, N, d, d, torch.float32, "simt")}))
