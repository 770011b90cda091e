"""Per-chunk pipeline timeline of the tensor-core prefill (CTA 0,0) via the debug trace hook."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2501_02573_b200 import _lib, ops

EV = ["-", "dS_issue", "O_issue", "P_done", "K_done", "O_stored", "dS_loaded", "S_published", "-", "-",
      "mma1_full_ok", "mma1_issued", "epi1_ok", "tma_load_issue", "st_full_ok", "-"]


def main(mode="full", B=8, H=32, N=8192, d=128, cta=0):
    lib = _lib.load()
    lib.linattn_debug_set_trace.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(16 * 4096, dtype=torch.int64, device="cuda")
    buf[15 * 4096] = int(cta)   # which (b*h) CTA to trace
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q)
    l2 = ops.log2_gamma([0.99] * H, True, "cuda")
    fn = (lambda: ops.prefill(q, k, v, l2)) if mode == "full" else (lambda: ops.state_pass(k, v, l2))
    fn(); torch.cuda.synchronize()
    lib.linattn_debug_set_trace(buf.data_ptr())
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    lib.linattn_debug_set_trace(None)
    print(f"{mode}: kernel {e0.elapsed_time(e1) * 1e3:.1f} us")
    t = buf.view(16, 4096).cpu().numpy().astype(np.int64)
    t0 = t.copy()
    n = (N + 63) // 64
    t = t[:, :n]
    base = t[1, 0]
    lo, hi = min(10, n - 1), max(min(n - 2, 100), 1)
    per = np.diff(t[1, lo:hi + 1])
    print(f"chunk period (dS issue to dS issue): median {np.median(per):.0f} cyc")
    for e in [1, 2, 3, 4, 5, 6, 7, 10, 11, 12, 13, 14]:
        rel = t[e, lo:hi] - t[1, lo:hi]
        if np.any(t[e, :n] != 0):
            print(f"  {EV[e]:26s} rel. to dS issue of same chunk: median {np.median(rel):8.0f}")
    nb = B * H * ((d + 127) // 128)
    st, en, sm = t0[8, :nb], t0[9, :nb], t0[0, :nb]
    live = st > 0                      # balanced launches run fewer CTAs (one per SM) than units
    st, en, sm = st[live], en[live], sm[live]
    nb = int(live.sum())
    t_min = st.min()
    print(f"CTAs {nb}: start span {(st.max() - t_min) / 1e3:.1f} us, end span {(en.min() - t_min) / 1e3:.1f}.."
          f"{(en.max() - t_min) / 1e3:.1f} us; CTA duration median {np.median(en - st) / 1e3:.1f} us "
          f"(min {np.min(en - st) / 1e3:.1f}, max {np.max(en - st) / 1e3:.1f})")
    order = np.argsort(st)
    late = order[148:]
    if len(late):
        print(f"  2nd-wave CTAs: start {np.median(st[late] - t_min) / 1e3:.1f} us, duration median "
              f"{np.median(en[late] - st[late]) / 1e3:.1f} us; 1st wave duration median "
              f"{np.median(en[order[:148]] - st[order[:148]]) / 1e3:.1f} us")
    for c in range(0, min(n, 4)):
        print("  chunk", c, " ".join(f"{EV[e]}={t[e, c] - base}" for e in [1, 2, 3, 4, 5, 6, 7, 10, 11, 12, 13, 14] if t[e, c]))


if __name__ == "__main__":
    shape = dict(zip("BHN", map(int, sys.argv[3].split(",")))) if len(sys.argv) > 3 else {}
    main(sys.argv[1] if len(sys.argv) > 1 else "full", cta=int(sys.argv[2]) if len(sys.argv) > 2 else 0, **shape)
