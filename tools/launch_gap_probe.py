"""Dev probe: configs[1] prefill timed back-to-back, one at a time (idle GPU before each), from a
CUDA graph, and the host cost per call -- where does the bench-vs-ncu gap come from?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
B, H, N, d = 8, 32, 8192, 128
q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
out = torch.empty_like(v)
l2 = ops.log2_gamma([1 - 2 ** (-5 - 10 * h / 31) for h in range(H)], True, "cuda")
f = lambda: ops.prefill(q, k, v, l2, out=out)
for _ in range(5): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(100): f()
e1.record(); torch.cuda.synchronize()
print(f"back-to-back: {e0.elapsed_time(e1) / 100 * 1e3:.1f} us")
ts = []
for _ in range(20):
    torch.cuda.synchronize(); time.sleep(0.002)
    e0.record(); f(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort(); print(f"isolated: median {ts[10]:.1f} us, min {ts[0]:.1f}")
t = time.perf_counter()
for _ in range(200): f()
h = (time.perf_counter() - t) / 200 * 1e6
torch.cuda.synchronize()
print(f"host time per call (enqueue): {h:.1f} us")
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    f(); torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20): f()
torch.cuda.current_stream().wait_stream(s)
g.replay(); torch.cuda.synchronize()
e0.record()
for _ in range(5): g.replay()
e1.record(); torch.cuda.synchronize()
print(f"graph of 20: {e0.elapsed_time(e1) / 100 * 1e3:.1f} us per launch")
