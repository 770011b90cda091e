"""Per-chunk timeline of the 3xTF32 prefill (fp32 parity mode) for CTA (0,0,0) via the debug
trace hook.  Needs a library built with -DTF32_TRACE=1:

    tools/build_variant.sh tft -DTF32_TRACE=1
    LINATTN_LIB=build/var/tft.so python tools/trace_tf32.py [B H N d]

Runs the plain grid (LINATTN_BALANCE=0): the traced CTA walks one (b*h, dv tile) unit."""
import ctypes, os, sys
os.environ["LINATTN_BALANCE"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2501_02573_b200 import _lib, ops

EV = {0: "state: dS ready", 1: "state: S updated", 2: "state: O ready", 3: "state: published",
      4: "state: O loaded", 5: "MMA: dS issued", 6: "MMA: Oi issued", 7: "MMA: MMA1 issued",
      8: "MMA: Ox issued", 9: "mask done", 10: "prepA (lo parts) done", 11: "prepB (K', Vlo) done",
      12: "TMA K|V issued", 13: "MMA loop top"}


def main(B=8, H=32, N=8192, d=128):
    lib = _lib.load()
    lib.linattn_debug_set_trace.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(16 * 4096, dtype=torch.int64, device="cuda")
    q = torch.randn(B, H, N, d, device="cuda")
    k, v = torch.randn_like(q), torch.randn_like(q)
    l2 = ops.log2_gamma([0.99] * H, True, "cuda")
    fn = lambda: ops.prefill(q, k, v, l2, kernel="tf32", seq_split=1)   # noqa: E731
    fn(); torch.cuda.synchronize()
    lib.linattn_debug_set_trace(buf.data_ptr())
    fn(); torch.cuda.synchronize()
    lib.linattn_debug_set_trace(None)
    t = buf.view(16, 4096).cpu().numpy().astype(np.int64)
    n = (N + 31) // 32
    t = t[:, :n]
    lo, hi = 20, n - 20
    per = np.diff(t[5, lo:hi + 1])
    print(f"chunk period (dS issue to dS issue): median {np.median(per):.0f} cyc  p10 {np.percentile(per, 10):.0f}"
          f"  p90 {np.percentile(per, 90):.0f}")
    for e in sorted(EV):
        if np.any(t[e] != 0):
            rel = t[e, lo:hi] - t[5, lo:hi]
            print(f"  {EV[e]:24s} rel. to dS issue of same chunk: median {np.median(rel):8.0f}  "
                  f"p10 {np.percentile(rel, 10):8.0f}  p90 {np.percentile(rel, 90):8.0f}")


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:5]))
