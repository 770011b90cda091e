"""Dev check of the 3xTF32 prefill kernel: parity against the f64 oracle on small shapes and
timing of the configs[1] shape in fp32 against the FFMA kernel (same process, CUDA events)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import linattn_oracle as orc  # noqa: E402
from paper_2501_02573_b200 import ops  # noqa: E402

dev = "cuda"
torch.cuda.set_device(0)
worst = 0.0
for (B, H, N, dk, dv, seed) in [(1, 1, 32, 32, 128, 0), (1, 2, 100, 64, 64, 1), (2, 3, 257, 128, 128, 2),
                                (1, 2, 1000, 128, 200, 3), (1, 1, 64, 4, 8, 4), (2, 2, 513, 96, 36, 5)]:
    b, c, v = orc.gen_inputs(B, H, N, dk, dv, np.float32, seed)
    gam = [[0.0, 0.9, 0.99, 1.0][h % 4] for h in range(H)]
    ref = orc.oracle_attn(b, c, v, gam, True)
    l2 = ops.log2_gamma(gam, True, dev)
    t = [torch.from_numpy(x).to(dev) for x in (b, c, v)]
    s_out = torch.zeros(B, H, dk, dv, device=dev)
    out = ops.prefill(*t, l2, kernel="tf32", s_out=s_out, seq_split=1)
    torch.cuda.synchronize()
    err = orc.max_rel_error(out.cpu().numpy(), ref)
    ref_o, ref_s = orc.seeded_blocked_attn(b, c, v, gam, True)
    serr = orc.max_rel_error(s_out.cpu().numpy(), ref_s)
    so = ops.state_pass(t[1], t[2], l2, kernel="tf32")
    sperr = orc.max_rel_error(so.cpu().numpy(), ref_s)
    worst = max(worst, err, serr, sperr)
    print(f"B={B} H={H} N={N} dk={dk} dv={dv}: out {err:.2e} s_out {serr:.2e} state_pass {sperr:.2e}", flush=True)
print("worst", worst)
# more (b, h) units than SMs with a partly filled last wave: balanced persistent launch
for (B, H, N, dk, dv) in [(1, 150, 300, 64, 128), (2, 100, 257, 128, 128), (1, 160, 1000, 32, 256)]:
    b, c, v = orc.gen_inputs(B, H, N, dk, dv, np.float32, 9)
    gam = [[0.0, 0.9, 0.99, 1.0, 0.5][h % 5] for h in range(H)]
    ref, ref_s = orc.seeded_blocked_attn(b, c, v, gam, True)
    t = [torch.from_numpy(x).to(dev) for x in (b, c, v)]
    s_out = torch.zeros(B, H, dk, dv, device=dev)
    out = ops.prefill(*t, ops.log2_gamma(gam, True, dev), kernel="tf32", s_out=s_out)
    print(f"balanced B={B} H={H} N={N} dk={dk} dv={dv}: out {orc.max_rel_error(out.cpu().numpy(), ref):.2e} "
          f"s_out {orc.max_rel_error(s_out.cpu().numpy(), ref_s):.2e}", flush=True)

B, H, N, d = 8, 32, 8192, 128
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn(B, H, N, d, device=dev, generator=g) for _ in range(3))
l2 = ops.log2_gamma([1 - 2.0 ** (-5 - 10 * h / 31) for h in range(H)], True, dev)
out = torch.empty_like(v)
for kern in ("tf32", "simt", "tf32"):
    for _ in range(3):
        ops.prefill(q, k, v, l2, out=out, kernel=kern)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ops.prefill(q, k, v, l2, out=out, kernel=kern)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{kern}: configs[1] fp32 {ms:.3f} ms, {B * H * N * 16 * d / ms / 1e6:.0f} GB/s", flush=True)
ref_tf = ops.prefill(q, k, v, l2, kernel="tf32")
ref_si = ops.prefill(q, k, v, l2, kernel="simt")
print("tf32 vs simt at full size:", orc.max_rel_error(ref_tf.cpu().numpy(), ref_si.cpu().numpy()))
