"""Dev timing of the split state pass (phase A) at the 8-GPU configs[4] slice, by sub-split m."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
B, H, N, d = 1, 32, 16384, 128
q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
l2 = ops.log2_gamma([1 - 2 ** (-5 - 10 * h / 31) for h in range(H)], True, "cuda")
def timeit(f, it=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3
loc = ops.state_pass_segmented(k, v, l2, 4096, m=1, nseg=4)
r = {}
for segs in (1, 2, 4, 8):
    sl = N // segs
    r[f"statepass_{segs}seg"] = timeit(lambda: ops.state_pass_segmented(k, v, l2, sl, m=1, nseg=segs))
r["prefix"] = timeit(lambda: ops.segment_prefix(loc, (4096, 1), 4096, 4, l2, N))
r["empty_launch_like_small_op"] = timeit(lambda: ops.prefix_combine(loc[:2], [N, N], 1, l2))
print(json.dumps(r))
