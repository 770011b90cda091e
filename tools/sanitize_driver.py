"""Small launches of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02573_b200 import ops  # noqa: E402

torch.manual_seed(0)
for (B, H, N, dk, dv) in [(1, 2, 300, 128, 128), (1, 1, 200, 64, 64), (1, 1, 130, 256, 512)]:
    q = torch.randn(B, H, N, dk, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn(B, H, N, dv, device="cuda", dtype=torch.bfloat16)
    l2 = ops.log2_gamma([0.9] * H, True, "cuda")
    s_out = torch.empty(B, H, dk, dv, device="cuda")
    ops.prefill(q, k, v, l2, s_out=s_out)                      # tensor-core kernel
    ops.prefill(q, k, v, l2, seq_split=3)                      # split: state pass + seeded segments
    ops.prefill(q.float(), k.float(), v.float(), l2, kernel="simt")
    st = torch.zeros(B, H, dk, dv, device="cuda")
    ops.decode_step(q[:, :, 0].contiguous(), k[:, :, 0].contiguous(), v[:, :, 0].contiguous(), st, l2)
    ops.prefix_combine(torch.stack([s_out, s_out]), [N, N], 1, l2)
# more units than SMs: the balanced persistent schedule (head -> tail state hand-off)
H = torch.cuda.get_device_properties(0).multi_processor_count + 5
for dk in (128, 64):
    q = torch.randn(1, H, 300, dk, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn(1, H, 300, 128, device="cuda", dtype=torch.bfloat16)
    l2 = ops.log2_gamma([0.9] * H, True, "cuda")
    ops.prefill(q, k, v, l2, s_in=torch.zeros(1, H, dk, 128, device="cuda"),
                s_out=torch.empty(1, H, dk, 128, device="cuda"))
# dk = 256 balanced schedule over two-CTA clusters (80 pairs > 74 co-resident)
q = torch.randn(1, 40, 200, 256, device="cuda", dtype=torch.bfloat16)
k = torch.randn_like(q)
v = torch.randn(1, 40, 200, 512, device="cuda", dtype=torch.bfloat16)
ops.prefill(q, k, v, ops.log2_gamma([0.9] * 40, True, "cuda"), s_out=torch.empty(1, 40, 256, 512, device="cuda"))
# any head width on the tensor cores (padded DK instantiations, dv not a multiple of 32 / 64),
# with initial and end states, the state pass and the in-device split
for (B, H, N, dk, dv) in [(2, 3, 333, 96, 72), (1, 2, 200, 200, 40), (1, 1, 150, 24, 8)]:
    q = torch.randn(B, H, N, dk, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn(B, H, N, dv, device="cuda", dtype=torch.bfloat16)
    l2 = ops.log2_gamma([0.9] * H, True, "cuda")
    ops.prefill(q, k, v, l2, s_in=torch.zeros(B, H, dk, dv, device="cuda"),
                s_out=torch.empty(B, H, dk, dv, device="cuda"), kernel="tc")
    ops.state_pass(k, v, l2, kernel="tc")
    ops.prefill(q, k, v, l2, seq_split=2, kernel="tc")
# fp32 parity mode on the tensor cores (3xTF32) and the row recurrence
q = torch.randn(2, 3, 300, 128, device="cuda")
k = torch.randn_like(q)
v = torch.randn(2, 3, 300, 128, device="cuda")
l2 = ops.log2_gamma([0.9] * 3, True, "cuda")
ops.prefill(q, k, v, l2, s_out=torch.empty(2, 3, 128, 128, device="cuda"), kernel="tf32")
ops.recurrent(q, k, v, l2, s_out=torch.empty(2, 3, 128, 128, device="cuda"))
torch.cuda.synchronize()
print("sanitize driver done")
