import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
B, H, N, d = [int(x) for x in sys.argv[1].split(",")]
q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
l2 = ops.log2_gamma([1 - 2 ** (-5 - 10 * h / max(1, H - 1)) for h in range(H)], True, "cuda")
plan = ops.seq_plan(B, H, N, d, d)
print("plan", plan, flush=True)
seg, nseg, m, sub = plan
t = time.time()
loc = ops.state_pass_segmented(k, v, l2, seg, m=m, nseg=nseg - 1)
torch.cuda.synchronize(); print("phase A ok", time.time() - t, flush=True)
o = ops.prefill_segmented(q, k, v, l2, seg, loc=loc, loc_geom=(seg, m))
torch.cuda.synchronize(); print("phase B ok", time.time() - t, flush=True)
o = ops.prefill(q, k, v, l2)
torch.cuda.synchronize(); print("auto ok", time.time() - t, flush=True)
