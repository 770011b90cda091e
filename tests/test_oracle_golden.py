"""Pin the CPU oracle (oracle/linattn_oracle.py) to the reference's own outputs.

golden.npz was produced by importing the reference package itself
(tests/golden/make_golden.py).  If /root/reference is present (build
container), the oracle is additionally checked against the live reference.
"""

import os
import sys

import numpy as np
import pytest

from oracle import linattn_oracle as orc
from la_helpers import FIXTURES, fixture_case

REF_SRC = "/root/reference/pkg/src"


@pytest.mark.parametrize("name", FIXTURES)
def test_fixtures_known_answers(golden, name):
    b, c, v, gamma, decay, expected = fixture_case(golden, name)
    out = orc.oracle_attn(b, c, v, gamma, decay)
    np.testing.assert_allclose(out[0, 0], expected, atol=1e-12)            # conftest.py:7-51 values
    np.testing.assert_allclose(out, golden[f"fx_{name}_oracle"], atol=1e-12)
    blk = orc.blocked_attn(b, c, v, gamma, decay, block=64)
    np.testing.assert_allclose(blk, golden[f"fx_{name}_tlb"], atol=1e-12)
    row, _ = orc.row_recurrence(b[0, 0], c[0, 0], v[0, 0], gamma[0], decay)
    np.testing.assert_allclose(row, golden[f"fx_{name}_row"][0, 0], atol=1e-12)


def _grid_case(golden, i):
    bt, hd, n, r, d, g, decay, bits = golden[f"grid_{i}_cfg"]
    dtype = np.float64 if int(bits) == 64 else np.float32
    b, c, v = orc.gen_inputs(int(bt), int(hd), int(n), int(r), int(d), dtype, 2026)
    insum = np.array([b.astype(np.float64).sum(), c.astype(np.float64).sum(), v.astype(np.float64).sum()])
    np.testing.assert_array_equal(insum, golden[f"grid_{i}_insum"])  # generator drift guard
    return b, c, v, [float(g)] * int(hd), bool(decay), dtype


def test_grid_oracle_and_blocked(golden):
    for i in range(int(golden["grid_count"])):
        b, c, v, gamma, decay, dtype = _grid_case(golden, i)
        ref = golden[f"grid_{i}_oracle"]
        out = orc.oracle_attn(b, c, v, gamma, decay, out_dtype=dtype)
        if dtype == np.float64:
            np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))
        else:
            np.testing.assert_array_equal(out, ref)  # same f64 math, same cast
        blk = orc.blocked_attn(b, c, v, gamma, decay, block=64)
        tol = 1e-10 if dtype == np.float64 else 1e-3  # reference tolerances (verify.py:14)
        assert orc.max_rel_error(blk, golden[f"grid_{i}_tlb"]) <= tol * 1e-2
        assert orc.max_rel_error(blk, ref) <= tol
        if f"grid_{i}_row" in golden:
            row = np.stack([np.stack([orc.row_recurrence(b[x, h], c[x, h], v[x, h], gamma[h], decay,
                                                         dtype=np.float64)[0]
                                      for h in range(b.shape[1])]) for x in range(b.shape[0])])
            assert orc.max_rel_error(row, golden[f"grid_{i}_row"]) <= tol
            assert orc.max_rel_error(row, ref) <= tol


def test_per_head_gamma(golden):
    out = orc.oracle_attn(golden["ph_b"], golden["ph_c"], golden["ph_v"], list(golden["ph_gamma"]), True)
    np.testing.assert_allclose(out, golden["ph_oracle"], atol=1e-12)


def test_bf16_cases_regenerate(golden):
    for i in range(int(golden["bf_count"])):
        bt, hd, n, r, d = (int(x) for x in golden[f"bf_{i}_cfg"])
        b, c, v = (orc.bf16_round(x) for x in orc.gen_inputs(bt, hd, n, r, d, np.float32, 7))
        insum = np.array([b.astype(np.float64).sum(), c.astype(np.float64).sum(), v.astype(np.float64).sum()])
        np.testing.assert_array_equal(insum, golden[f"bf_{i}_insum"])
        if n * r <= 300 * 64:
            out = orc.oracle_attn(b, c, v, list(golden[f"bf_{i}_gamma"]), True)
            assert orc.max_rel_error(out, golden[f"bf_{i}_oracle"]) <= 1e-6


def test_sp_algebra_matches_oracle():
    # per-segment scan + exclusive gamma prefix == oracle
    b, c, v = orc.gen_inputs(1, 1, 203, 5, 7, np.float64, 3)
    for gamma in (0.0, 0.9, 1.0):
        ref = orc.oracle_attn(b, c, v, [gamma], True)[0, 0]
        for parts in (1, 2, 4, 8):
            out = orc.sp_blocked_attn(b[0, 0], c[0, 0], v[0, 0], gamma, parts, True, block=16)
            assert orc.max_rel_error(out, ref) <= 1e-13


def test_decode_continuity_matches_oracle():
    # prefill end state of 256 tokens + 44 decode steps == oracle on 300 tokens (Appendix B.6)
    b, c, v = orc.gen_inputs(1, 2, 300, 6, 5, np.float64, 11)
    gammas = [0.97, 1.0]
    ref = orc.oracle_attn(b, c, v, gammas, True)
    state = np.stack([[orc.segment_end_state(c[0, h, :256], v[0, h, :256], gammas[h]) for h in range(2)]])
    out, _ = orc.decode_steps(b[:, :, 256:], c[:, :, 256:], v[:, :, 256:], state, gammas)
    assert orc.max_rel_error(out, ref[:, :, 256:]) <= 1e-13


def test_block_size_invariance():
    b, c, v = orc.gen_inputs(1, 2, 33, 4, 6, np.float64, 35)
    base = orc.blocked_attn(b, c, v, [0.9, 0.9], True, block=1)
    for bs in (2, 7, 32, 33, 38):
        assert orc.max_rel_error(orc.blocked_attn(b, c, v, [0.9, 0.9], True, block=bs), base) <= 1e-10


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present (GPU box)")
def test_oracle_against_live_reference():
    sys.path.insert(0, REF_SRC)
    try:
        import linattn
        from linattn import MethodId
        from linattn.bench import gen_inputs
        for (bt, hd, n, r, d, g, decay) in [(2, 3, 65, 8, 5, 0.9, True), (1, 2, 130, 16, 16, 0.0, True),
                                            (1, 1, 40, 3, 3, 1.0, False)]:
            inp = gen_inputs(bt, hd, n, r, d, np.float64, 9, decay, g)
            b, c, v = orc.gen_inputs(bt, hd, n, r, d, np.float64, 9)
            assert np.array_equal(b, inp.b) and np.array_equal(v, inp.v)
            ref = linattn.oracle_attn(inp, mem_cap=0)
            np.testing.assert_allclose(orc.oracle_attn(b, c, v, inp.gamma, decay), ref, atol=1e-12)
            tlb, _ = linattn.run_method(MethodId.TWO_LEVEL_BLOCK, inp)
            assert orc.max_rel_error(orc.blocked_attn(b, c, v, inp.gamma, decay), tlb) <= 1e-14
    finally:
        sys.path.remove(REF_SRC)
