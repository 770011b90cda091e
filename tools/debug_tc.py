"""Diagnostics for the tensor-core prefill: per-config / per-chunk error maps vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import linattn_oracle as orc
from paper_2501_02573_b200 import ops


def run(B, H, N, dk, dv, gam, seed=7, kernel="tc"):
    b, c, v = (orc.bf16_round(x) for x in orc.gen_inputs(B, H, N, dk, dv, np.float32, seed))
    ref = orc.oracle_attn(b, c, v, gam, True)
    l2 = ops.log2_gamma(gam, True, "cuda")
    t = lambda x: torch.from_numpy(x).cuda().to(torch.bfloat16)
    s_out = torch.zeros(B, H, dk, dv, device="cuda")
    out = ops.prefill(t(b), t(c), t(v), l2, s_out=s_out, kernel=kernel).float().cpu().numpy()
    sref = np.stack([[orc.segment_end_state(c[x, h], v[x, h], gam[h]) for h in range(H)] for x in range(B)])
    err = np.abs(out - ref) / np.abs(ref).max()
    serr = orc.max_rel_error(s_out.cpu().numpy(), sref)
    print(f"B{B} H{H} N{N} dk{dk} dv{dv} g{gam}: out err {err.max():.3e}  state err {serr:.3e}")
    nch = (N + 63) // 64
    for h in range(H):
        per_chunk = [err[:, h, 64 * i:64 * (i + 1)].max() for i in range(nch)]
        print(f"   head {h} chunks: " + " ".join(f"{x:.1e}" for x in per_chunk))
    if err.max() > 2e-2:
        x, h, tt, dd = np.unravel_index(np.argmax(err), err.shape)
        print(f"   worst at b{x} h{h} t{tt} d{dd}: got {out[x,h,tt,dd]:.4f} want {ref[x,h,tt,dd]:.4f}")
        e0 = err[0, h]
        print("   err by t (first 70):", " ".join(f"{e0[i].max():.0e}" for i in range(min(70, N))))
        print("   err by d:", " ".join(f"{e0[:, j].max():.0e}" for j in range(dv)))


torch.manual_seed(0)
run(1, 1, 64, 64, 64, [1.0])
run(1, 1, 64, 64, 64, [0.0])
run(1, 1, 64, 64, 64, [0.9])
run(1, 1, 64, 128, 128, [1.0])
run(1, 1, 128, 64, 64, [1.0])
run(1, 1, 128, 64, 64, [0.9])
run(1, 1, 128, 128, 128, [0.9])
run(1, 1, 44, 64, 64, [1.0])
run(1, 4, 300, 64, 64, [0.0, 0.5, 0.97, 1.0])
run(1, 2, 513, 128, 128, [0.96875, 1 - 2 ** -12])
