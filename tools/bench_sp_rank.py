"""Per-rank cost of sequence-parallel prefill at the 8-GPU configs[4] slice (1 x 32 x 16384 x 128)
vs the plain in-device split prefill of the same slice (what the all-gather path adds)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_02573_b200 import ops
from paper_2501_02573_b200.sp import CudaBackend
B, H, N, d = 1, 32, 16384, 128
q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
l2 = ops.log2_gamma([1 - 2 ** (-5 - 10 * h / 31) for h in range(H)], True, "cuda")
be = CudaBackend()
s_in = torch.zeros(B, H, d, d, device="cuda")
gathered = torch.zeros(8, B, H, d, d, device="cuda")


def rank_path():
    data, end = be.local_states(k, v, l2)
    si = be.prefix_combine(gathered, [N] * 8, 7, l2)
    be.prefill(q, k, v, l2, si, data)


def timeit(f, it=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


print(json.dumps({"plain_split_us": timeit(lambda: ops.prefill(q, k, v, l2)),
                  "sp_rank_path_us": timeit(rank_path),
                  "plan": ops.seq_plan(B, H, N, d, d)}))

# the same rank path replayed from a CUDA graph (no host gaps between the five launches)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    rank_path()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        rank_path()
torch.cuda.current_stream().wait_stream(s)
print(json.dumps({"sp_rank_path_graph_us": timeit(g.replay)}))
data, end = be.local_states(k, v, l2)
print(json.dumps({"phaseA_and_prefix_us": timeit(lambda: be.local_states(k, v, l2)),
                  "phaseB_us": timeit(lambda: be.prefill(q, k, v, l2, s_in, data))}))
