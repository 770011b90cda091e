"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``linattn`` from /root/reference/pkg/src (read-only; nothing is
copied) and writes ``tests/golden/golden.npz``.  The GPU box never needs the
reference: tests read the committed npz.

Contents (all outputs are produced by the reference's own functions):
  * ``fx_<name>_*``: the canonical fixtures EX-A..EX-E (reference
    tests/conftest.py:7-51) with their analytic expected values, plus the
    reference oracle_attn / two-level-block / row-based outputs on them.
  * ``grid_<i>_*``: a sample of the reference verify grid (verify.py:16-19)
    at f64 and f32, inputs regenerated from gen_inputs (bench.py:77-84)
    and pinned by an input checksum; outputs of oracle_attn, two-level-block,
    block-based and row-based.
  * ``ph_*``: per-head gamma case (test_kernels.py:195-201 style).
  * ``bf_<i>_*``: bf16-rounded gen_inputs(seed=7) at GPU-sized shapes (pinned
    by checksum) with the reference oracle output, for the device parity tests.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _bf16_round(a: np.ndarray) -> np.ndarray:
    """Round f32 to the nearest bf16 (ties to even) and return it as f32."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def main(path=os.path.join(HERE, "golden.npz")):
    sys.path.insert(0, REF_SRC)
    import linattn
    from linattn import MethodId, make_inputs, oracle_attn, run_method
    from linattn.bench import gen_inputs

    out = {}

    # --- canonical fixtures (reference tests/conftest.py:7-51) -------------
    rng3 = np.random.default_rng(3)
    d_b, d_c, d_v = rng3.standard_normal((1, 4)), rng3.standard_normal((1, 4)), rng3.standard_normal((1, 3))
    rng4 = np.random.default_rng(4)
    e_b, e_c, e_v = rng4.standard_normal((5, 3)), rng4.standard_normal((5, 3)), rng4.standard_normal((5, 2))
    fixtures = {
        "ex_a": ([[2.0], [3.0]], [[1.0], [4.0]], [[5.0], [6.0]], 1.0, False, [[10.0], [87.0]]),
        "ex_b": ([[2.0], [3.0]], [[1.0], [4.0]], [[5.0], [6.0]], 0.5, True, [[10.0], [79.5]]),
        "ex_c": (np.ones((3, 1)), np.ones((3, 1)), [[1.0, 0.0], [0.0, 1.0], [2.0, 2.0]], 1.0, False,
                 [[1.0, 0.0], [1.0, 1.0], [3.0, 3.0]]),
        "ex_d": (d_b, d_c, d_v, 1.0, False, float(d_b[0] @ d_c[0]) * d_v),
        "ex_e": (e_b, e_c, e_v, 0.0, True, (e_b * e_c).sum(axis=1, keepdims=True) * e_v),
    }
    for name, (b, c, v, g, decay, expected) in fixtures.items():
        inp = make_inputs(b, c, v, gamma=g, decay=decay)
        out[f"fx_{name}_b"] = inp.b
        out[f"fx_{name}_c"] = inp.c
        out[f"fx_{name}_v"] = inp.v
        out[f"fx_{name}_gamma"] = np.array(inp.gamma)
        out[f"fx_{name}_decay"] = np.array(decay)
        out[f"fx_{name}_expected"] = np.asarray(expected, dtype=np.float64)
        out[f"fx_{name}_oracle"] = oracle_attn(inp)
        out[f"fx_{name}_tlb"] = run_method(MethodId.TWO_LEVEL_BLOCK, inp)[0]
        out[f"fx_{name}_row"] = run_method(MethodId.ROW_BASED, inp)[0]

    # --- sample of the reference verify grid (verify.py:16-19) -------------
    grid = []
    for decay in (False, True):
        for (bt, hd) in ((1, 1), (2, 3)):
            for n in (1, 2, 3, 5, 16, 31, 32, 33, 64, 257):
                for (r, d) in ((1, 1), (3, 3), (8, 8), (32, 32)):
                    for g in (0.0, 0.5, 0.9, 1.0):
                        grid.append((bt, hd, n, r, d, g, decay))
    sel = np.random.default_rng(2026).choice(len(grid), size=48, replace=False)
    cases = [grid[i] for i in sorted(sel)]
    cases += [(2, 3, 257, 32, 32, 0.9, True), (1, 1, 257, 8, 8, 0.0, True),
              (2, 3, 33, 8, 8, 1.0, True), (1, 1, 64, 32, 32, 0.5, True)]
    for i, (bt, hd, n, r, d, g, decay) in enumerate(cases):
        dtype = np.float64 if i % 2 == 0 else np.float32
        inp = gen_inputs(bt, hd, n, r, d, dtype, 2026, decay, g)
        out[f"grid_{i}_cfg"] = np.array([bt, hd, n, r, d, g, float(decay), 64 if dtype == np.float64 else 32])
        out[f"grid_{i}_insum"] = np.array([inp.b.astype(np.float64).sum(), inp.c.astype(np.float64).sum(),
                                           inp.v.astype(np.float64).sum()])
        out[f"grid_{i}_oracle"] = oracle_attn(inp, mem_cap=0)
        out[f"grid_{i}_tlb"] = run_method(MethodId.TWO_LEVEL_BLOCK, inp)[0]
        if inp.v.nbytes <= 100_000:  # keep the npz small: the big cases carry oracle + tlb only
            out[f"grid_{i}_bb"] = run_method(MethodId.BLOCK_BASED, inp)[0]
            out[f"grid_{i}_row"] = run_method(MethodId.ROW_BASED, inp)[0]
            out[f"grid_{i}_rec"] = run_method(MethodId.RECURSION, inp)[0]
    out["grid_count"] = np.array(len(cases))

    # --- per-head gamma (test_kernels.py:195-201 style) ---------------------
    inp = gen_inputs(1, 2, 12, 3, 3, np.float64, seed=44, decay=True)
    inp.gamma = [0.3, 0.95]
    out["ph_b"], out["ph_c"], out["ph_v"] = inp.b, inp.c, inp.v
    out["ph_gamma"] = np.array(inp.gamma)
    out["ph_oracle"] = oracle_attn(inp)

    # --- bf16-representable GPU-sized cases ----------------------------------
    bf_cases = [
        # (B, H, N, r, d, gammas)
        (1, 4, 300, 64, 64, [0.0, 0.5, 0.97, 1.0]),
        (1, 2, 513, 128, 128, [0.96875, 1.0 - 2.0 ** -12]),
        (1, 1, 192, 256, 128, [0.99]),
    ]
    for i, (bt, hd, n, r, d, gs) in enumerate(bf_cases):
        inp = gen_inputs(bt, hd, n, r, d, np.float32, 7, True, 1.0)
        inp.b, inp.c, inp.v = _bf16_round(inp.b), _bf16_round(inp.c), _bf16_round(inp.v)
        inp.gamma = list(gs)
        # inputs are regenerated by the tests (gen_inputs seed 7 + bf16 rounding); pin them by checksum
        out[f"bf_{i}_cfg"] = np.array([bt, hd, n, r, d])
        out[f"bf_{i}_insum"] = np.array([inp.b.astype(np.float64).sum(), inp.c.astype(np.float64).sum(),
                                         inp.v.astype(np.float64).sum()])
        out[f"bf_{i}_gamma"] = np.array(gs)
        ref = linattn.oracle_attn(linattn.AttnInputs(
            b=inp.b.astype(np.float64), c=inp.c.astype(np.float64), v=inp.v.astype(np.float64),
            gamma=list(gs), decay=True))
        out[f"bf_{i}_oracle"] = ref.astype(np.float32)
    out["bf_count"] = np.array(len(bf_cases))

    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
