"""Dev probe: prefill time vs head count around one wave (dk=256/dv=512 clusters, or dk=128)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
dk, dv, N = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "256,512,16384").split(","))
for H in [int(h) for h in (sys.argv[2] if len(sys.argv) > 2 else "16,32,36,37,40,48,64").split(",")]:
    q = torch.randn(1, H, N, dk, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn(1, H, N, dv, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(v)
    l2 = ops.log2_gamma([0.99] * H, True, "cuda")
    kw = {} if os.environ.get("PROBE_AUTO") else {"seq_split": 1}
    f = lambda: ops.prefill(q, k, v, l2, out=out, **kw)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"H={H:3d} ms={ms:.4f} per-head us={ms * 1e3 / H:.2f}", flush=True)
