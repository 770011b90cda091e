import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
B, H, N, d, seg, m, nseg, mode = [int(x) for x in sys.argv[1].split(",")]
q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
l2 = ops.log2_gamma([1 - 2 ** (-5 - 10 * h / max(1, H - 1)) for h in range(H)], True, "cuda")
torch.cuda.synchronize()
t = time.time()
if mode == 0:
    loc = ops.state_pass_segmented(k, v, l2, seg, m=m, nseg=nseg)
elif mode == 1:
    ops.prefill(q, k, v, l2)
elif mode == 2:
    ops.state_pass(k, v, l2)
torch.cuda.synchronize(); print(sys.argv[1], "ok", round(time.time() - t, 4), flush=True)
