"""Dump the 3xTF32 kernel's first-chunk intermediates (CTA 0) and compare with numpy."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_02573_b200 import _lib, ops  # noqa: E402

lib = _lib.load()
dump = torch.zeros(36864, device="cuda")
lib.linattn_debug_set_tf32_dump.argtypes = [ctypes.c_void_p]
lib.linattn_debug_set_tf32_dump(dump.data_ptr())
rng = np.random.default_rng(0)
N, dk, dv = 32, 128, 128
q, k, v = (rng.standard_normal((1, 1, N, d)).astype(np.float32) for d in (dk, dk, dv))
g = 0.9
l2 = ops.log2_gamma([g], True, "cuda")
out = ops.prefill(*(torch.from_numpy(x).cuda() for x in (q, k, v)), l2, kernel="tf32", seq_split=1)
torch.cuda.synchronize()
lib.linattn_debug_set_tf32_dump(None)
D = dump.cpu().numpy()
print("pw", D[:5], "expect", [g ** i for i in range(5)])
P = D[64:64 + 1024].reshape(32, 32)     # P^T[s][t]
Pe = k[0, 0] @ q[0, 0].T
print("P^T rel err", np.abs(P - Pe).max() / np.abs(Pe).max(), "sample", P[0, :4], Pe[0, :4])


def unswz(buf, rows, cols, b32=False):
    """[cols/32 boxes][rows][32] with 128B swizzle (16B chunks ^ row%8, or 32B granules ^ row%4)."""
    out = np.zeros((rows, cols), np.float32)
    for b in range(cols // 32):
        for r in range(rows):
            for j in range(8):
                pos = ((((j >> 1) ^ (r & 3)) << 1) | (j & 1)) if b32 else (j ^ (r & 7))
                src = b * 1024 + r * 32 + pos * 4
                out[r, b * 32 + 4 * j: b * 32 + 4 * j + 4] = buf[src: src + 4]
    return out


Ks = unswz(D[20480:24576], 32, 128)
Vs = unswz(D[24576:28672], 32, 128, True)
Kp = unswz(D[28672:32768], 32, 128, True)
Vl = unswz(D[32768:36864], 32, 128, True)
print("K smem vs k (trunc):", np.abs(Ks - k[0, 0]).max())
print("V smem vs v (trunc):", np.abs(Vs - v[0, 0]).max())
w = np.array([g ** (31 - s) for s in range(32)], np.float32)
print("K'hi vs w k:", np.abs(Kp - w[:, None] * k[0, 0]).max())
print("Vhi+Vlo vs v:", np.abs(Vs + Vl - v[0, 0]).max())
dS = D[2048:2048 + 16384].reshape(128, 128)    # dS^T[d][i]
dSe = (v[0, 0].T @ (w[:, None] * k[0, 0]))
print("dS^T rel err", np.abs(dS - dSe).max() / np.abs(dSe).max(), "sample", dS[0, :4], dSe[0, :4])
print("out sample", out[0, 0, :2, :4].cpu().numpy())
