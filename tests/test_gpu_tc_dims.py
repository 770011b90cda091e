"""Tensor-core prefill at every dk <= 256 and dv with 16-byte rows (bf16), not just the
dk in {64, 128, 256} / dv % 64 == 0 of the benched configs.

The reference accepts any rank r and value dim d (verify.py:16-19, kernels.py:139-166); here a
head of width dk runs on the kernel for the next DK in {64, 128, 256} with the Q/K boxes past dk
zero-filled by TMA, and V boxes past dv zero-filled / output stores clipped.  Checked against
the seeded f64 blocked oracle within the bf16 bar (2e-2), including s_in / s_out (external
states are [B, H, dk, dv], not padded), the in-device sequence split and the balanced schedule.
"""

import numpy as np
import pytest
import torch

from oracle import linattn_oracle as orc

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02573_b200 import _lib, ops
    _lib.load()
    return ops


def dev(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def test_dispatch_takes_tensor_cores(ops):
    for dk, dv in [(8, 8), (32, 64), (96, 96), (192, 512), (200, 40), (256, 512), (128, 72)]:
        assert ops.prefill_kernel_name(dk, dv, torch.bfloat16) == "prefill_tc", (dk, dv)
    for dk, dv in [(264, 64), (12, 64), (64, 12)]:          # > 256, or rows not a multiple of 16 B
        assert ops.prefill_kernel_name(dk, dv, torch.bfloat16) == "prefill_simt", (dk, dv)


def _check(ops, B, H, N, dk, dv, gam, seed, split=None):
    rng = np.random.default_rng(seed)
    b, c, v = (orc.bf16_round(x) for x in orc.gen_inputs(B, H, N, dk, dv, np.float32, seed))
    s0 = rng.standard_normal((B, H, dk, dv)).astype(np.float32) * 0.05
    ref, ref_s = orc.seeded_blocked_attn(b, c, v, gam, True, s0.astype(np.float64), block=64)
    l2 = ops.log2_gamma(gam, True, "cuda")
    s_out = torch.full((B, H, dk, dv), float("nan"), device="cuda")
    kw = {} if split is None else {"seq_split": split}
    out = ops.prefill(dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16), l2,
                      s_in=dev(s0), s_out=s_out, kernel="tc", **kw)
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16, (B, H, N, dk, dv)
    assert orc.max_rel_error(s_out.cpu().numpy(), ref_s) <= 5e-3, (B, H, N, dk, dv)
    # state pass alone (K4): same end state
    st = ops.state_pass(dev(c, torch.bfloat16), dev(v, torch.bfloat16), l2, kernel="tc")
    _, ref_z = orc.seeded_blocked_attn(b, c, v, gam, True, np.zeros_like(s0, dtype=np.float64), block=64)
    assert orc.max_rel_error(st.cpu().numpy(), ref_z) <= 5e-3, ("state_pass", B, H, N, dk, dv)


@pytest.mark.parametrize("dk,dv", [(8, 8), (32, 64), (32, 100 - 4), (48, 136), (96, 96), (96, 200),
                                   (120, 128), (136, 64), (192, 512), (200, 40), (248, 264)])
def test_general_dims(ops, dk, dv):
    H = 3
    _check(ops, 2, H, 333, dk, dv, [0.0, 0.9, 1.0][:H], seed=dk * 1000 + dv)


@pytest.mark.parametrize("dk,dv", [(32, 64), (96, 128), (192, 256)])
def test_general_dims_sequence_split(ops, dk, dv):
    """Few heads, long N: the in-device two-phase split (local states are [.., dk, dv] too)."""
    assert ops.seq_plan(1, 2, 8192, dk, dv)[1] > 1
    _check(ops, 1, 2, 8192, dk, dv, [0.99, 1 - 2.0 ** -12], seed=7 + dk)


@pytest.mark.parametrize("dk,dv", [(32, 128), (96, 64)])
def test_general_dims_balanced(ops, dk, dv):
    """More (b, h) units than SMs with a poorly filled last wave: the balanced persistent schedule
    (hand-off states hold the padded DK rows internally)."""
    H = torch.cuda.get_device_properties(0).multi_processor_count + 7
    gam = [[0.5, 0.9, 0.99, 1.0][h % 4] for h in range(H)]
    _check(ops, 1, H, 200, dk, dv, gam, seed=11 + dk)


@pytest.mark.parametrize("dt,dk,dv", [(torch.bfloat16, 12, 20), (torch.float32, 3, 5), (torch.float32, 6, 128)])
def test_recurrent_route_odd_rows(dt, dk, dv):
    """b200-recurrent (row-based semantics, kernels.py:93-106) on rows that are not a multiple of
    16 bytes: zero-padded to one and run by the single-launch scan kernel (no per-token loop)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_02573_b200 as la
    from paper_2501_02573_b200 import _lib
    b, c, v = orc.gen_inputs(2, 3, 150, dk, dv, np.float32, dk + dv)
    if dt == torch.bfloat16:
        b, c, v = (orc.bf16_round(x) for x in (b, c, v))
    gam = [0.5, 0.95, 1.0]
    ref = orc.oracle_attn(b, c, v, gam, True)
    inp = la.make_inputs(dev(b, dt), dev(c, dt), dev(v, dt), gamma=gam, decay=True)
    before = _lib.launch_count()
    out, _ = la.run_method(la.MethodId.B200_RECURRENT, inp)
    torch.cuda.synchronize()
    assert _lib.launch_count() - before < 10          # one scan launch, not 150 decode steps
    tol = TOL_BF16 if dt == torch.bfloat16 else 1e-4
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= tol
