"""Per-chunk timeline of the dk=256 TMEM-state kernel (CTA 0,0,0) via the debug trace hook."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2501_02573_b200 import _lib, ops

EV = {0: "state start", 1: "st_done", 2: "P^T ld done", 3: "S-upd issued", 4: "O issued", 5: "MMA1 issued(c)",
      6: "ox_scaled", 7: "V' done", 8: "O drained", 9: "TMA issue", 10: "MMA warp ready", 11: "P^T start",
      12: "V' start", 14: "P^T done", 13: "O ready"}


def main(mode="full", B=4, H=16, N=16384, dk=256, dv=512):
    lib = _lib.load()
    lib.linattn_debug_set_trace.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(16 * 4096, dtype=torch.int64, device="cuda")
    q = torch.randn(B, H, N, dk, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn(B, H, N, dv, device="cuda", dtype=torch.bfloat16)
    l2 = ops.log2_gamma([0.99] * H, True, "cuda")
    fn = (lambda: ops.prefill(q, k, v, l2, seq_split=1)) if mode == "full" else (lambda: ops.state_pass(k, v, l2))
    fn(); torch.cuda.synchronize()
    lib.linattn_debug_set_trace(buf.data_ptr())
    fn(); torch.cuda.synchronize()
    lib.linattn_debug_set_trace(None)
    t = buf.view(16, 4096).cpu().numpy().astype(np.int64)
    n = (N + 63) // 64
    t = t[:, :n]
    lo, hi = 20, n - 20
    per = np.diff(t[3, lo:hi + 1])
    print(f"{mode}: chunk period (S-upd issue to S-upd issue): median {np.median(per):.0f} cyc")
    for e in sorted(EV):
        if np.any(t[e] != 0):
            rel = t[e, lo:hi] - t[3, lo:hi]
            print(f"  {EV[e]:18s} rel. to S-upd issue of same chunk: median {np.median(rel):8.0f}  p10 {np.percentile(rel, 10):8.0f}  p90 {np.percentile(rel, 90):8.0f}")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["full"]))
