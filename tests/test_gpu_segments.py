"""Sequence segments on one device: the split plan, the segmented C ABI and the SP pieces.

The algebra is the reference recursion cross term (kernels.py:185-189) applied across
segments; every result is checked against the f64 oracle (oracle/linattn_oracle.py) at
the tolerances of test_gpu_parity.py (bf16 tensor cores 2e-2, fp32 FFMA 1e-4).
"""

import numpy as np
import pytest
import torch

from oracle import linattn_oracle as orc

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
TOL_F32 = 1e-4


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02573_b200 import _lib, ops
    _lib.load()
    return ops


def dev(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def _inputs(B, H, N, dk, dv, seed, gam):
    b, c, v = orc.gen_inputs(B, H, N, dk, dv, np.float32, seed)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    return b, c, v, orc.oracle_attn(b, c, v, gam, True)


def test_seq_plan_shapes(ops):
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    seg, nseg, m, sub = ops.seq_plan(1, 32, 131072, 128, 128)        # configs[4] on one GPU
    assert nseg > 1 and seg % 64 == 0 and nseg * 32 <= sms and sub % 64 == 0
    assert ops.seq_plan(8, 32, 8192, 128, 128)[1] == 1                # configs[1]: units fill the SMs
    # fp32 parity mode (FFMA kernel, 64-wide dv tiles, 2 CTAs/SM) splits too: configs[0] shape
    seg, nseg, m, _ = ops.seq_plan(1, 8, 2048, 64, 64, torch.float32)
    assert nseg > 1 and 8 * nseg <= 2 * sms and seg % 64 == 0


@pytest.mark.parametrize("dk,dv", [(128, 128), (64, 128), (256, 256)])
def test_auto_split_matches_oracle(ops, dk, dv):
    gam = [1 - 2.0 ** -5, 1 - 2.0 ** -12]
    b, c, v, ref = _inputs(1, 2, 4096, dk, dv, 31, gam)
    l2 = ops.log2_gamma(gam, True, "cuda")
    q, k, vv = dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16)
    s_out = torch.empty(1, 2, dk, dv, device="cuda")
    out = ops.prefill(q, k, vv, l2, s_out=s_out)                     # library plan (split)
    one = ops.prefill(q, k, vv, l2, seq_split=1)                      # single pass
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16
    assert orc.max_rel_error(one.float().cpu().numpy(), ref) <= TOL_BF16
    ref_s = np.stack([[orc.segment_end_state(c[0, h], v[0, h], gam[h]) for h in range(2)]])
    assert orc.max_rel_error(s_out.cpu().numpy(), ref_s) <= 5e-3


@pytest.mark.parametrize("seg_len,m", [(256, 1), (256, 2), (256, 3), (512, 4), (64, 1)])
@pytest.mark.parametrize("mode", ["tc", "simt", "tf32"])
def test_segmented_geometries(ops, seg_len, m, mode):
    """Ragged N, empty sub-segments (256/3 -> 128+128+0), s_in seeding and the end state."""
    B, H, N, d = 2, 3, 1000, 64 if mode == "simt" else 128
    gam = [0.0, 0.97, 1.0]
    b, c, v = orc.gen_inputs(B, H, N, d, d, np.float32, 32)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    s0 = np.random.default_rng(5).standard_normal((B, H, d, d)).astype(np.float32) * 0.1
    ref, ref_s = orc.seeded_blocked_attn(b, c, v, gam, True, s0.astype(np.float64), block=64)
    dt, tol = (torch.bfloat16, TOL_BF16) if mode == "tc" else (torch.float32, TOL_F32)
    kernel = mode
    l2 = ops.log2_gamma(gam, True, "cuda")
    q, k, vv = dev(b, dt), dev(c, dt), dev(v, dt)
    nseg = -(-N // seg_len)
    loc = ops.state_pass_segmented(k, vv, l2, seg_len, m=m, nseg=nseg, kernel=kernel)
    s_out = torch.empty(B, H, d, d, device="cuda")
    out = ops.prefill_segmented(q, k, vv, l2, seg_len, loc=loc, loc_geom=(seg_len, m), s_in=dev(s0),
                                s_out=s_out, kernel=kernel)
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= tol
    assert orc.max_rel_error(s_out.cpu().numpy(), ref_s) <= (5e-3 if mode == "tc" else 1e-5)
    # the state at N from the local states equals the seeded end state
    end = ops.state_at(loc, (seg_len, m), N, l2, N, s_in=dev(s0))
    assert orc.max_rel_error(end.cpu().numpy(), ref_s) <= (5e-3 if mode == "tc" else 1e-5)
    # inclusive prefixes at every segment end, then the one-read-per-segment seeded prefill
    incl = ops.segment_prefix(loc, (seg_len, m), seg_len, nseg, l2, N)
    for p in (0, nseg // 2, nseg - 1):
        hi = min(N, (p + 1) * seg_len)
        want = np.stack([[orc.segment_end_state(c[x, h, :hi], v[x, h, :hi], gam[h]) for h in range(H)]
                         for x in range(B)])
        assert orc.max_rel_error(incl[p].cpu().numpy(), want) <= (5e-3 if mode == "tc" else 1e-5)
    out2 = ops.prefill_segmented(q, k, vv, l2, seg_len, loc=incl[:-1] if nseg > 1 else None, loc_geom=(seg_len, 1),
                                 inclusive=True, s_in=dev(s0), kernel=kernel)
    assert orc.max_rel_error(out2.float().cpu().numpy(), ref) <= tol


@pytest.mark.parametrize("parts", [2, 3, 8])
def test_sp_pieces_loopback(ops, parts):
    """Multi-GPU SP with the all-gather replaced by a stack of per-rank end states."""
    from paper_2501_02573_b200.sp import CudaBackend, segment_bounds
    gam = [1 - 2.0 ** -4, 1 - 2.0 ** -14, 0.0]
    b, c, v, ref = _inputs(1, 3, 3000, 128, 128, 33, gam)
    l2 = ops.log2_gamma(gam, True, "cuda")
    be = CudaBackend()
    bounds = segment_bounds(3000, parts)
    lens = [hi - lo for lo, hi in bounds]
    segs = [[dev(x[:, :, lo:hi], torch.bfloat16) for x in (b, c, v)] for lo, hi in bounds]
    locals_ = [be.local_states(k, vv, l2) for _, k, vv in segs]
    ends = torch.stack([end for _, end in locals_])
    outs = []
    for r, ((q, k, vv), (data, _)) in enumerate(zip(segs, locals_)):
        s_in = be.prefix_combine(ends, lens, r, l2) if r > 0 else None
        outs.append(be.prefill(q, k, vv, l2, s_in, data))
    got = torch.cat(outs, dim=2).float().cpu().numpy()
    assert orc.max_rel_error(got, ref) <= TOL_BF16


def test_split_causality_and_linearity(ops):
    """configs[4]-shaped heads at N=32768 (split by the plan): bitwise causality and linearity."""
    torch.manual_seed(1)
    B, H, N, d = 1, 8, 32768, 128
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q)
    gam = [1 - 2 ** (-5 - 10 * h / (H - 1)) for h in range(H)]
    l2 = ops.log2_gamma(gam, True, "cuda")
    assert ops.seq_plan(B, H, N, d, d)[1] > 1
    o = ops.prefill(q, k, v, l2)
    assert torch.equal(ops.prefill(q, k, (2 * v).contiguous(), l2), 2 * o)
    k2 = k.clone()
    k2[:, :, 30000:] = torch.randn_like(k2[:, :, 30000:])
    assert torch.equal(ops.prefill(q, k2, v, l2)[:, :, :30000], o[:, :, :30000])
    one = ops.prefill(q, k, v, l2, seq_split=1)
    assert orc.max_rel_error(o.float().cpu().numpy(), one.float().cpu().numpy()) <= TOL_BF16
    # sampled head against the oracle over the last 4096 tokens, seeded with the exact prefix state
    h = 3
    qq, kk, vv = (x[0, h].float().cpu().numpy().astype(np.float64) for x in (q, k, v))
    s_pre = orc.segment_end_state(kk[:N - 4096], vv[:N - 4096], gam[h])
    ref, _ = orc.seeded_blocked_attn(qq[None, None, N - 4096:], kk[None, None, N - 4096:],
                                     vv[None, None, N - 4096:], [gam[h]], True, s_pre[None, None], block=64)
    assert orc.max_rel_error(o[0, h, N - 4096:].float().cpu().numpy(), ref[0, 0]) <= TOL_BF16


def test_cuda_graph_capture_split_and_decode(ops):
    """The split prefill (stream-ordered pool workspace) and the decode step replay from a CUDA graph."""
    torch.manual_seed(2)
    B, H, N, d = 1, 4, 8192, 128
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q)
    l2 = ops.log2_gamma([0.99, 0.999, 0.5, 1.0], True, "cuda")
    assert ops.seq_plan(B, H, N, d, d)[1] > 1
    out = torch.empty_like(v)
    st = torch.zeros(B, H, d, d, device="cuda")
    qd, kd, vd = (x[:, :, 0].contiguous() for x in (q, k, v))
    od = torch.empty_like(vd)
    want = ops.prefill(q, k, v, l2).clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ops.prefill(q, k, v, l2, out=out)          # warm-up outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            ops.prefill(q, k, v, l2, out=out)
            ops.decode_step(qd, kd, vd, st, l2, out=od)
    torch.cuda.current_stream().wait_stream(s)
    out.zero_()
    st.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    # two replays of the decode step from S = 0: S = (gamma + 1) k^T v
    s2 = torch.zeros_like(st)
    ops.decode_step(qd, kd, vd, s2, l2)
    ops.decode_step(qd, kd, vd, s2, l2)
    assert torch.allclose(st, s2, rtol=1e-6, atol=1e-6)


def test_long_context_gamma_near_one(ops):
    """SURVEY.md 7 "decay numerics": gamma in [1-1e-5, 1-1e-7] at N = 131072 (configs[4] length).

    fp32-rounded gamma would put ~4e-3 relative error on gamma^n there; the kernels take log2(gamma)
    derived in f64.  The split prefill's last 2048 tokens are checked against an f64 reference
    seeded with the exact f64 prefix state.
    """
    torch.manual_seed(3)
    B, H, N, d = 1, 2, 131072, 64
    gam = [1 - 1e-5, 1 - 1e-7]
    q = (torch.randn(B, H, N, d, device="cuda") * 0.25).to(torch.bfloat16)
    k = (torch.randn(B, H, N, d, device="cuda") * 0.25).to(torch.bfloat16)
    v = torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16)
    l2 = ops.log2_gamma(gam, True, "cuda")
    assert ops.seq_plan(B, H, N, d, d)[1] > 1
    o = ops.prefill(q, k, v, l2)
    T = 2048
    for h in range(H):
        kk = k[0, h].double().cpu().numpy()
        vv = v[0, h].double().cpu().numpy()
        w = np.exp((N - T - 1 - np.arange(N - T)) * np.log(gam[h]))        # f64 gamma^(L-1-t)
        s_pre = (kk[:N - T] * w[:, None]).T @ vv[:N - T]
        qq = q[0, h, N - T:].double().cpu().numpy()
        ref, _ = orc.seeded_blocked_attn(qq[None, None], kk[None, None, N - T:], vv[None, None, N - T:],
                                         [gam[h]], True, s_pre[None, None], block=64)
        assert orc.max_rel_error(o[0, h, N - T:].float().cpu().numpy(), ref[0, 0]) <= TOL_BF16


@pytest.mark.parametrize("B,H,dk,dv", [(2, 80, 128, 128), (1, 75, 64, 256), (3, 53, 128, 192),
                                       (1, 40, 256, 512), (3, 30, 256, 256)])
@pytest.mark.parametrize("N", [1, 64, 200, 1000])
def test_balanced_schedule(ops, B, H, dk, dv, N):
    """More units than SMs (not a whole number of waves) runs the balanced persistent schedule:
    sequence heads publish their end state to the next CTA's range (dk = 256: to the same cluster
    rank of the next two-CTA cluster's range).  Checked with s_in seeding
    and s_out against the seeded f64 blocked oracle, gamma in {0, 1} included."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    units = B * H * -(-dv // 128)
    assert units > sms and units % sms != 0           # the balanced path is the one under test
    gam = [0.0, 1.0] + [1 - 2.0 ** (-3 - (h % 12)) for h in range(H - 2)]
    b, c, v = orc.gen_inputs(B, H, N, dk, dv, np.float32, 40 + N)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    s0 = np.random.default_rng(N).standard_normal((B, H, dk, dv)).astype(np.float32) * 0.05
    ref, ref_s = orc.seeded_blocked_attn(b, c, v, gam, True, s0.astype(np.float64), block=64)
    l2 = ops.log2_gamma(gam, True, "cuda")
    q, k, vv = dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16)
    s_out = torch.full((B, H, dk, dv), float("nan"), device="cuda")
    out = ops.prefill(q, k, vv, l2, s_in=dev(s0), s_out=s_out)
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16
    assert orc.max_rel_error(s_out.cpu().numpy(), ref_s) <= 5e-3
    # repeated launches reuse the pooled workspace (flags re-zeroed per launch)
    again = ops.prefill(q, k, vv, l2, s_in=dev(s0))
    assert torch.equal(again, out)


@pytest.mark.parametrize("kernel", ["simt", "tf32"])
@pytest.mark.parametrize("B,H,N,dk,dv", [(3, 53, 300, 128, 128), (2, 80, 1000, 64, 96), (1, 150, 65, 32, 64),
                                         (1, 149, 2000, 128, 128)])
def test_balanced_schedule_fp32(ops, B, H, N, dk, dv, kernel):
    """The balanced persistent schedules of the fp32 kernels (FFMA: more 64-wide units than
    resident CTAs; 3xTF32: more 128-wide units than SMs with a poorly filled last wave): fp32
    parity with s_in seeding and s_out at the 1e-4 bar."""
    gam = [0.0, 1.0] + [1 - 2.0 ** (-3 - (h % 12)) for h in range(H - 2)]
    b, c, v = orc.gen_inputs(B, H, N, dk, dv, np.float32, 60 + N)
    s0 = np.random.default_rng(N).standard_normal((B, H, dk, dv)).astype(np.float32) * 0.05
    ref, ref_s = orc.seeded_blocked_attn(b, c, v, gam, True, s0.astype(np.float64), block=64)
    l2 = ops.log2_gamma(gam, True, "cuda")
    s_out = torch.full((B, H, dk, dv), float("nan"), device="cuda")
    out = ops.prefill(dev(b), dev(c), dev(v), l2, s_in=dev(s0), s_out=s_out, kernel=kernel)
    assert orc.max_rel_error(out.cpu().numpy(), ref) <= TOL_F32
    assert orc.max_rel_error(s_out.cpu().numpy(), ref_s) <= TOL_F32


def test_batch_heads_beyond_grid_limit(ops):
    """More than 65535 (batch, head) units: ops splits the batch into launches of <= 65535 units
    (the C ABI rejects larger ones); results equal independent smaller calls bitwise."""
    B, H, N, d = 2100, 32, 3, 16
    g = torch.Generator(device="cuda").manual_seed(5)
    l2 = ops.log2_gamma([0.5 + 0.015 * h for h in range(H)], True, "cuda")
    for dt, kernel in ((torch.bfloat16, "auto"), (torch.float32, "simt")):
        q, k, v = (torch.randn(B, H, N, d, device="cuda", dtype=dt, generator=g) for _ in range(3))
        s0 = torch.randn(B, H, d, d, device="cuda", generator=g)
        s_out = torch.empty_like(s0)
        out = ops.prefill(q, k, v, l2, s_in=s0, s_out=s_out, kernel=kernel)
        for b0, b1 in ((0, 1000), (1000, B)):
            so = torch.empty_like(s0[b0:b1])
            part = ops.prefill(q[b0:b1].contiguous(), k[b0:b1].contiguous(), v[b0:b1].contiguous(), l2,
                               s_in=s0[b0:b1].contiguous(), s_out=so, kernel=kernel)
            assert torch.equal(part, out[b0:b1]) and torch.equal(so, s_out[b0:b1])
        rec = ops.recurrent(q, k, v, l2)
        assert torch.equal(rec[1000:1010], ops.recurrent(q[1000:1010].contiguous(), k[1000:1010].contiguous(),
                                                          v[1000:1010].contiguous(), l2))
        ref = orc.oracle_attn(q[2099:].float().cpu().numpy(), k[2099:].float().cpu().numpy(),
                              v[2099:].float().cpu().numpy(), [0.5 + 0.015 * h for h in range(H)], True)
        assert orc.max_rel_error(rec[2099:].float().cpu().numpy(), ref) <= (TOL_F32 if dt == torch.float32 else TOL_BF16)


@pytest.mark.parametrize("dt,kernel", [(torch.bfloat16, "auto"), (torch.float32, "simt"), (torch.float32, "tf32")])
def test_state_pass_split(ops, dt, kernel):
    """Few (b, h) units: the state pass runs every segment in parallel and scans them (the same
    plan as the prefill split); the end state matches the oracle and the unsplit prefill's s_out."""
    gam = [0.0, 0.97, 1 - 2.0 ** -12]
    b, c, v = orc.gen_inputs(1, 3, 5000, 128, 128, np.float32, 77)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    l2 = ops.log2_gamma(gam, True, "cuda")
    assert ops.seq_plan(1, 3, 5000, 128, 128, dt, kernel)[1] > 1
    s = ops.state_pass(dev(c, dt), dev(v, dt), l2, kernel=kernel)
    ref = np.stack([[orc.segment_end_state(c[0, h], v[0, h], gam[h]) for h in range(3)]])
    assert orc.max_rel_error(s.cpu().numpy(), ref) <= (2e-3 if dt == torch.bfloat16 else 1e-5)
    s1 = torch.empty_like(s)
    ops.prefill(dev(b, dt), dev(c, dt), dev(v, dt), l2, s_out=s1, kernel=kernel, seq_split=1)
    assert orc.max_rel_error(s.cpu().numpy(), s1.cpu().numpy()) <= (2e-3 if dt == torch.bfloat16 else 1e-5)


@pytest.mark.parametrize("seed", range(12))
def test_sp_fuzz(ops, seed):
    """Sequence parallelism with the all-gather replaced by a stack: random rank counts, uneven
    (possibly tiny) segments, head dims incl. dk=256, bf16 tensor cores and the fp32 FFMA backend."""
    from paper_2501_02573_b200.sp import CudaBackend
    rng = np.random.default_rng(700 + seed)
    P = int(rng.choice([2, 3, 5, 8]))
    dk, dv = [(64, 64), (128, 128), (128, 256), (256, 512)][int(rng.integers(0, 4))]
    B, H = int(rng.choice([1, 2])), int(rng.choice([1, 3]))
    cuts = np.sort(rng.choice(np.arange(1, 4000), size=P - 1, replace=False))
    N = int(cuts[-1] + rng.integers(1, 800))
    bounds = list(zip([0] + cuts.tolist(), cuts.tolist() + [N]))
    gam = [float(rng.choice([0.0, 0.9, 1 - 2.0 ** -10, 1.0])) for _ in range(H)]
    fp32 = bool(rng.integers(0, 2)) and dk <= 128
    dt, tol, kernel = (torch.float32, TOL_F32, ["simt", "tf32"][seed % 2]) if fp32 else (torch.bfloat16, TOL_BF16, "auto")
    b, c, v = orc.gen_inputs(B, H, N, dk, dv, np.float32, 800 + seed)
    if not fp32:
        b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    ref, _ = orc.seeded_blocked_attn(b, c, v, gam, True, None, block=64)
    l2 = ops.log2_gamma(gam, True, "cuda")
    be = CudaBackend(kernel)
    lens = [hi - lo for lo, hi in bounds]
    segs = [[dev(x[:, :, lo:hi], dt) for x in (b, c, v)] for lo, hi in bounds]
    locals_ = [be.local_states(k, vv, l2) for _, k, vv in segs]
    ends = torch.stack([end for _, end in locals_])
    outs = [be.prefill(q, k, vv, l2, be.prefix_combine(ends, lens, r, l2) if r > 0 else None, data)
            for r, ((q, k, vv), (data, _)) in enumerate(zip(segs, locals_))]
    got = torch.cat(outs, dim=2).float().cpu().numpy()
    assert orc.max_rel_error(got, ref) <= tol, (P, lens, dk, dv, fp32)
