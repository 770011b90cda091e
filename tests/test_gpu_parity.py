"""Device parity: every device method against the oracle / golden vectors.

Tolerances (north star; max-norm relative error, verify.py:22-24):
  * bf16 tensor-core path ("b200-chunked", "b200-seqpar"): <= 2e-2
  * fp32 parity mode ("b200-chunked-f32", "b200-recurrent"): <= 1e-4 vs the f64 oracle
All calls go through the C ABI (liblinattn_b200.so) via the package API.
"""

import numpy as np
import pytest
import torch

from la_helpers import FIXTURES, fixture_case
from oracle import linattn_oracle as orc

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
TOL_F32 = 1e-4


@pytest.fixture(scope="module")
def la():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_02573_b200 as la
    from paper_2501_02573_b200 import _lib
    _lib.load()  # fail loudly if the library is missing
    return la


def dev(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def test_library_loaded_and_launches(la):
    from paper_2501_02573_b200 import _lib
    before = _lib.launch_count()
    inp = la.make_inputs(dev(np.ones((4, 2))), dev(np.ones((4, 2))), dev(np.ones((4, 3))))
    la.run_method(la.MethodId.B200_CHUNKED_F32, inp)
    torch.cuda.synchronize()
    assert _lib.launch_count() > before


@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("method", ["b200-chunked-f32", "b200-chunked", "b200-recurrent", "b200-seqpar"])
def test_canonical_fixtures(la, golden, name, method):
    b, c, v, gamma, decay, expected = fixture_case(golden, name)
    inp = la.make_inputs(b, c, v, gamma=gamma, decay=decay)   # host f64 arrays, like the reference
    out, ops = la.run_method(la.MethodId.parse(method), inp)
    assert isinstance(out, np.ndarray) and out.dtype == np.float64 and ops > 0
    tol = TOL_BF16 if method in ("b200-chunked", "b200-seqpar") else TOL_F32
    if name in ("ex_a", "ex_b", "ex_c"):
        np.testing.assert_allclose(out[0, 0], expected, atol=1e-6)   # exact in bf16 and fp32
    else:
        assert orc.max_rel_error(out[0, 0], expected) <= tol


def _grid(golden, i):
    bt, hd, n, r, d, g, decay, bits = golden[f"grid_{i}_cfg"]
    dtype = np.float64 if int(bits) == 64 else np.float32
    b, c, v = orc.gen_inputs(int(bt), int(hd), int(n), int(r), int(d), dtype, 2026)
    return b, c, v, [float(g)] * int(hd), bool(decay)


def test_reference_grid_f32_mode(la, golden):
    worst = 0.0
    for i in range(int(golden["grid_count"])):
        b, c, v, gamma, decay = _grid(golden, i)
        out, _ = la.run_method(la.MethodId.B200_CHUNKED_F32, la.make_inputs(b, c, v, gamma, decay))
        err = orc.max_rel_error(out, golden[f"grid_{i}_oracle"])
        worst = max(worst, err)
        assert err <= TOL_F32, (i, err)
    print(f"f32 grid worst {worst:.2e}")


def test_reference_grid_bf16_tc(la, golden):
    for i in range(int(golden["grid_count"])):
        b, c, v, gamma, decay = _grid(golden, i)
        bq, cq, vq = (dev(orc.bf16_round(x), torch.bfloat16) for x in (b, c, v))
        inp = la.make_inputs(bq, cq, vq, gamma, decay)
        out, _ = la.run_method(la.MethodId.B200_CHUNKED, inp)
        ref = orc.oracle_attn(orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v), gamma, decay)
        assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16, i


@pytest.mark.parametrize("kernel", ["auto", "simt"])
def test_bf16_golden_cases(la, golden, kernel):
    from paper_2501_02573_b200 import ops
    for i in range(int(golden["bf_count"])):
        bt, hd, n, r, d = (int(x) for x in golden[f"bf_{i}_cfg"])
        b, c, v = (orc.bf16_round(x) for x in orc.gen_inputs(bt, hd, n, r, d, np.float32, 7))
        gam = list(golden[f"bf_{i}_gamma"])
        ref = golden[f"bf_{i}_oracle"]
        l2 = ops.log2_gamma(gam, True, "cuda")
        out = ops.prefill(dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16), l2,
                          kernel=kernel)
        assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16, (i, kernel)
        out32 = ops.prefill(dev(b), dev(c), dev(v), l2, kernel="simt")
        assert orc.max_rel_error(out32.cpu().numpy(), ref) <= TOL_F32, i


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 127, 129, 300])
@pytest.mark.parametrize("dk,dv", [(64, 64), (128, 128), (32, 48), (256, 128), (128, 256)])
def test_shapes_and_ragged(la, n, dk, dv):
    from paper_2501_02573_b200 import ops
    b, c, v = orc.gen_inputs(2, 3, n, dk, dv, np.float32, 5)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    gam = [0.0, 0.9, 1.0]
    ref = orc.oracle_attn(b, c, v, gam, True)
    l2 = ops.log2_gamma(gam, True, "cuda")
    out = ops.prefill(dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16), l2)
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16
    out32 = ops.prefill(dev(b), dev(c), dev(v), l2, kernel="simt")
    assert orc.max_rel_error(out32.cpu().numpy(), ref) <= TOL_F32


def test_binary_mask_and_per_head_gamma(la, golden):
    inp = la.make_inputs(golden["ph_b"], golden["ph_c"], golden["ph_v"], list(golden["ph_gamma"]), True)
    out, _ = la.run_method(la.MethodId.B200_CHUNKED_F32, inp)
    assert orc.max_rel_error(out, golden["ph_oracle"]) <= TOL_F32
    b, c, v = orc.gen_inputs(1, 2, 150, 16, 8, np.float64, 1)
    out, _ = la.run_method(la.MethodId.B200_CHUNKED_F32, la.make_inputs(b, c, v, [0.3, 0.5], decay=False))
    assert orc.max_rel_error(out, orc.oracle_attn(b, c, v, [1.0, 1.0], False)) <= TOL_F32


def test_state_out_and_state_pass(la):
    from paper_2501_02573_b200 import ops
    b, c, v = orc.gen_inputs(2, 2, 200, 64, 64, np.float32, 8)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    gam = [0.95, 1.0]
    l2 = ops.log2_gamma(gam, True, "cuda")
    ref = np.stack([[orc.segment_end_state(c[x, h], v[x, h], gam[h]) for h in range(2)] for x in range(2)])
    for kernel in ("auto", "simt"):
        for dt in (torch.bfloat16, torch.float32):
            k_sel = kernel if dt == torch.bfloat16 else "simt"
            # fp32-FFMA kernel: fp32 everywhere -> 1e-5.  Tensor-core kernel: the decayed keys
            # K' = gamma^(L-1-s) K are bf16 MMA operands -> bf16-level state error.
            tol = 2e-3 if ops.prefill_kernel_name(64, 64, dt, k_sel) == "prefill_tc" else 1e-5
            s = ops.state_pass(dev(c, dt), dev(v, dt), l2, kernel=k_sel)
            assert orc.max_rel_error(s.cpu().numpy(), ref) <= tol
            s_out = torch.empty_like(s)
            ops.prefill(dev(b, dt), dev(c, dt), dev(v, dt), l2, s_out=s_out, kernel=k_sel)
            assert orc.max_rel_error(s_out.cpu().numpy(), ref) <= tol


def test_prefix_combine(la):
    from paper_2501_02573_b200 import ops
    rng = np.random.default_rng(0)
    P, B, H, dk, dv = 5, 2, 3, 8, 12
    states = rng.standard_normal((P, B, H, dk, dv)).astype(np.float32)
    lens = [7, 0, 130, 1, 64]
    gam = [0.0, 0.97, 1.0]
    l2 = ops.log2_gamma(gam, True, "cuda")
    for rank in range(P):
        got = ops.prefix_combine(dev(states), lens, rank, l2).cpu().numpy()
        for h in range(H):
            want = orc.exclusive_prefix_states([states[p][:, h] for p in range(P)], lens, gam[h])[rank]
            np.testing.assert_allclose(got[:, h], want, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("parts", [1, 2, 3, 4])
def test_seqpar_loopback(la, parts):
    b, c, v = orc.gen_inputs(1, 4, 1000, 128, 128, np.float32, 12)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    gam = [1 - 2.0 ** -5, 1 - 2.0 ** -10, 1 - 2.0 ** -15, 0.5]
    inp = la.make_inputs(dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16), gam, True)
    out, _ = la.run_method(la.MethodId.B200_SEQPAR, inp, la.BlockParams(seq_parts=parts))
    assert orc.max_rel_error(out.float().cpu().numpy(), orc.oracle_attn(b, c, v, gam, True)) <= TOL_BF16


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_prefill_then_decode_continuity(la, dt):
    b, c, v = orc.gen_inputs(2, 3, 300, 64, 128, np.float32, 13)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    gam = [0.0, 0.97, 1.0]
    ref = orc.oracle_attn(b, c, v, gam, True)
    pre = la.make_inputs(dev(b[:, :, :256], dt), dev(c[:, :, :256], dt), dev(v[:, :, :256], dt), gam, True)
    out, state = la.prefill_with_state(pre, kernel="simt" if dt == torch.float32 else "auto")
    tol = TOL_F32 if dt == torch.float32 else TOL_BF16
    assert orc.max_rel_error(out.float().cpu().numpy(), ref[:, :, :256]) <= tol
    outs = [state.step(dev(b[:, :, i], dt), dev(c[:, :, i], dt), dev(v[:, :, i], dt)) for i in range(256, 300)]
    got = torch.stack(outs, dim=2).float().cpu().numpy()
    assert orc.max_rel_error(got, ref[:, :, 256:]) <= tol


def test_decode_steps_vs_oracle(la):
    from paper_2501_02573_b200 import ops
    rng = np.random.default_rng(3)
    B, H, dk, dv, T = 4, 3, 128, 128, 20
    s0 = rng.standard_normal((B, H, dk, dv))
    q, k, v = (rng.standard_normal((B, H, T, d)) for d in (dk, dk, dv))
    gam = [0.0, 0.9, 1.0]
    ref, ref_s = orc.decode_steps(q, k, v, s0, gam)
    st = dev(s0)
    l2 = ops.log2_gamma(gam, True, "cuda")
    outs = [ops.decode_step(dev(q[:, :, i]), dev(k[:, :, i]), dev(v[:, :, i]), st, l2) for i in range(T)]
    got = torch.stack(outs, 2).cpu().numpy()
    assert orc.max_rel_error(got, ref) <= TOL_F32
    assert orc.max_rel_error(st.cpu().numpy(), ref_s) <= TOL_F32


@pytest.mark.parametrize("dk,dv", [(3, 5), (64, 62), (128, 512), (128, 128), (64, 96), (32, 100), (256, 512)])
def test_decode_odd_shapes(la, dk, dv):
    """Few (b, h) states: the columns are split over CTAs (ragged last slice included)."""
    from paper_2501_02573_b200 import ops
    rng = np.random.default_rng(4)
    B, H = 2, 2
    s0 = rng.standard_normal((B, H, dk, dv))
    q, k, v = (rng.standard_normal((B, H, 1, d)) for d in (dk, dk, dv))
    ref, ref_s = orc.decode_steps(q, k, v, s0, [0.8, 1.0])
    st = dev(s0)
    o = ops.decode_step(dev(q[:, :, 0]), dev(k[:, :, 0]), dev(v[:, :, 0]), st,
                        ops.log2_gamma([0.8, 1.0], True, "cuda"))
    assert orc.max_rel_error(o.cpu().numpy(), ref[:, :, 0]) <= TOL_F32
    assert orc.max_rel_error(st.cpu().numpy(), ref_s) <= TOL_F32


def test_full_size_properties(la):
    """cfg2-shaped (B=8,H=32,N=8192,d=128) properties the oracle cannot check densely."""
    from paper_2501_02573_b200 import ops
    torch.manual_seed(0)
    B, H, N, d = 8, 32, 8192, 128
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    gam = [1 - 2.0 ** (-5 - 10 * h / (H - 1)) for h in range(H)]
    l2 = ops.log2_gamma(gam, True, "cuda")
    o = ops.prefill(q, k, v, l2)
    # linearity in V: scaling by 2 is exact in bf16 and fp32
    o2 = ops.prefill(q, k, (2 * v).contiguous(), l2)
    assert torch.equal(o2, 2 * o)
    # causality: perturbing the last 1000 tokens leaves the first 7168 outputs bitwise unchanged
    k2 = k.clone()
    k2[:, :, 7192:] = torch.randn_like(k2[:, :, 7192:])
    o3 = ops.prefill(q, k2, v, l2)
    assert torch.equal(o3[:, :, :7168], o[:, :, :7168])
    # sampled slices against the f64 oracle
    for (bi, h) in [(0, 0), (7, 31)]:
        ref = orc.oracle_attn(q[bi:bi + 1, h:h + 1].float().cpu().numpy(), k[bi:bi + 1, h:h + 1].float().cpu().numpy(),
                              v[bi:bi + 1, h:h + 1].float().cpu().numpy(), [gam[h]], True)
        assert orc.max_rel_error(o[bi, h].float().cpu().numpy(), ref[0, 0]) <= TOL_BF16
    # sequence split on one device agrees with the single pass (two-phase, 4 segments)
    inp = la.make_inputs(q[:1], k[:1], v[:1], gam, True)
    sp, _ = la.run_method(la.MethodId.B200_SEQPAR, inp, la.BlockParams(seq_parts=4))
    assert orc.max_rel_error(sp.float().cpu().numpy(), o[:1].float().cpu().numpy()) <= TOL_BF16


def test_cfg3_shape_small_n(la):
    """RetNet-shaped heads: dk=256, dv=512 (configs[2]) at a size the oracle can check."""
    from paper_2501_02573_b200 import ops
    b, c, v = orc.gen_inputs(1, 2, 257, 256, 512, np.float32, 14)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    gam = [1 - 2.0 ** -5, 1 - 2.0 ** -8]
    ref = orc.oracle_attn(b, c, v, gam, True)
    out = ops.prefill(dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16),
                      ops.log2_gamma(gam, True, "cuda"))
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16


@pytest.mark.parametrize("batch,heads,dt", [(3, 2, torch.bfloat16), (1, 5, torch.bfloat16), (2, 3, torch.float32)])
def test_host_tensor_pipeline(la, batch, heads, dt):
    """Host (pinned and pageable) torch tensors: piecewise H2D | kernel | D2H equals the device call."""
    b, c, v = orc.gen_inputs(batch, heads, 300, 64, 128, np.float32, 15)
    gam = [1 - 2.0 ** -(3 + h) for h in range(heads)]
    method = la.MethodId.B200_CHUNKED if dt == torch.bfloat16 else la.MethodId.B200_CHUNKED_F32
    hb, hc, hv = (torch.from_numpy(x).to(dt) for x in (b, c, v))
    want, _ = la.run_method(method, la.make_inputs(hb.cuda(), hc.cuda(), hv.cuda(), gam, True))
    pinned = [x.pin_memory() for x in (hb, hc, hv)]
    out = torch.empty(hv.shape, dtype=dt).pin_memory()
    got, ops = la.run_method(method, la.make_inputs(*pinned, gam, True), out=out)
    assert got is out and ops > 0 and torch.equal(got, want.cpu())
    got2, _ = la.run_method(method, la.make_inputs(hb, hc, hv, gam, True))
    assert torch.equal(got2, want.cpu())


def test_configs0_shape_fp32_and_bf16(la):
    """BASELINE configs[0]: B=1, H=8, N=2048, d=64, fp32, per-head gamma (the reference's own
    CPU blocking-vs-naive case): fp32 parity mode <= 1e-4 and the tensor-core path <= 2e-2
    against the f64 oracle, and the reference blocking route (oracle port) agrees too."""
    b, c, v = orc.gen_inputs(1, 8, 2048, 64, 64, np.float32, 2026)
    gam = [1 - 2.0 ** (-5 - h) for h in range(8)]
    ref = orc.oracle_attn(b, c, v, gam, True)
    out, ops_count = la.run_method(la.MethodId.B200_CHUNKED_F32, la.make_inputs(b, c, v, gam, True))
    assert out.dtype == np.float32 and orc.max_rel_error(out, ref) <= TOL_F32
    assert orc.max_rel_error(orc.blocked_attn(b, c, v, gam, True, block=64), ref) <= 1e-5
    auto = la.decode(la.make_inputs(b, c, v, gam, True))            # auto -> fp32 mode for f32 input
    assert orc.max_rel_error(auto, ref) <= TOL_F32
    bq, cq, vq = (orc.bf16_round(x) for x in (b, c, v))
    ref16 = orc.oracle_attn(bq, cq, vq, gam, True)
    out16, _ = la.run_method(la.MethodId.B200_CHUNKED,
                             la.make_inputs(*(dev(x, torch.bfloat16) for x in (bq, cq, vq)), gam, True))
    assert orc.max_rel_error(out16.float().cpu().numpy(), ref16) <= TOL_BF16


@pytest.mark.parametrize("dk,dv", [(128, 192), (64, 64), (256, 128)])
@pytest.mark.parametrize("decay", [True, False])
def test_split_binary_mask_and_partial_dv_tile(la, dk, dv, decay):
    """The library's own sequence split (B*H small) with a partial dv tile and the binary mask."""
    from paper_2501_02573_b200 import ops
    b, c, v = orc.gen_inputs(1, 2, 3000, dk, dv, np.float32, 41)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v) * 0.25
    gam = [0.5, 1.0]
    assert ops.seq_plan(1, 2, 3000, dk, dv)[1] > 1
    ref = orc.oracle_attn(b, c, v, gam if decay else [1.0, 1.0], decay)
    out = ops.prefill(dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16),
                      ops.log2_gamma(gam, decay, "cuda"))
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16


def test_run_bench_gpu_rows(la):
    """run_bench with CUDA-event timing and roofline columns (reference bench.py:87-125)."""
    cfg = la.BenchConfig(methods=[la.MethodId.B200_CHUNKED, la.MethodId.B200_CHUNKED_F32],
                         grid=[(1, 4, 1024, 64, 64), (2, 2, 333, 128, 128)], decay=True, repeats=3, warmup=1)
    rep = la.run_bench(cfg)
    assert len(rep.rows) == 4
    for r in rep.rows:
        assert r.status == "ok" and r.mean_s > 0 and r.opcount > 0 and r.gbps > 0 and 0 < r.frac_hbm < 1.5
    assert "PCG64" in rep.meta["generator"] and "CUDA events" in rep.meta["timing"]
    assert la.render_report(rep, "csv").count("\n") == 5


def test_unaligned_views_route_to_ffma_kernel(la):
    """A contiguous but 2-byte-offset view cannot be a TMA base: AUTO runs the FFMA kernel,
    an explicit tensor-core request raises the reference's UsageError."""
    from paper_2501_02573_b200 import ops
    B, H, N, d = 1, 2, 200, 64
    b, c, v = (orc.bf16_round(x) for x in orc.gen_inputs(B, H, N, d, d, np.float32, 17))
    gam = [0.9, 0.99]
    ref = orc.oracle_attn(b, c, v, gam, True)

    def unaligned(x):
        flat = torch.empty(x.size + 1, device="cuda", dtype=torch.bfloat16)
        view = flat[1:].view(x.shape)
        view.copy_(torch.from_numpy(x))
        assert view.data_ptr() % 16 != 0
        return view

    q, k, vv = unaligned(b), unaligned(c), unaligned(v)
    l2 = ops.log2_gamma(gam, True, "cuda")
    out = ops.prefill(q, k, vv, l2)
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16
    with pytest.raises(la.UsageError):
        ops.prefill(q, k, vv, l2, kernel="tc")


@pytest.mark.parametrize("decay", [True, False])
def test_dk256_lazy_normalisation_regimes(la, decay):
    """dk=256 keeps S = sig * T with a scalar sig per head; gamma = 0.5 renormalises every chunk,
    0.9 every few chunks, 0.99 / 0.9999 rarely or never, 0 always, 1 never (binary mask)."""
    from paper_2501_02573_b200 import ops
    gam = [0.5, 0.9, 0.99, 0.9999, 0.0, 1.0]
    b, c, v = (orc.bf16_round(x) for x in orc.gen_inputs(1, 6, 3000, 256, 256, np.float32, 19))
    v = orc.bf16_round(v * 0.25)
    ref = orc.oracle_attn(b, c, v, gam if decay else [1.0] * 6, decay)
    s_out = torch.empty(1, 6, 256, 256, device="cuda")
    out = ops.prefill(dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16),
                      ops.log2_gamma(gam, decay, "cuda"), s_out=s_out, seq_split=1)
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16
    ref_s = np.stack([[orc.segment_end_state(c[0, h], v[0, h], gam[h] if decay else 1.0) for h in range(6)]])
    assert orc.max_rel_error(s_out.cpu().numpy(), ref_s) <= 5e-3


@pytest.mark.parametrize("dk,dv,dt", [(128, 128, torch.float32), (64, 256, torch.bfloat16), (256, 128, torch.float32),
                                      (8, 12, torch.float32)])
def test_recurrent_scan_kernel(la, dk, dv, dt):
    """b200-recurrent = the reference row-based route in one launch (kernels.py:93-106)."""
    from paper_2501_02573_b200 import ops
    gam = [0.0, 0.93, 1.0]
    b, c, v = (orc.bf16_round(x) for x in orc.gen_inputs(2, 3, 333, dk, dv, np.float32, 21))
    ref = orc.oracle_attn(b, c, v, gam, True)
    out, opc = la.run_method(la.MethodId.B200_RECURRENT, la.make_inputs(dev(b, dt), dev(c, dt), dev(v, dt), gam, True))
    assert opc > 0
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= (TOL_F32 if dt == torch.float32 else TOL_BF16)
    # seeded state in / state out continues a sequence exactly like one pass
    l2 = ops.log2_gamma(gam, True, "cuda")
    if dv % 4 == 0:
        s_mid = torch.empty(2, 3, dk, dv, device="cuda")
        ops.recurrent(dev(b[:, :, :200], dt), dev(c[:, :, :200], dt), dev(v[:, :, :200], dt), l2, s_out=s_mid)
        tail = ops.recurrent(dev(b[:, :, 200:], dt), dev(c[:, :, 200:], dt), dev(v[:, :, 200:], dt), l2, s_in=s_mid)
        assert orc.max_rel_error(tail.float().cpu().numpy(), ref[:, :, 200:]) <= (TOL_F32 if dt == torch.float32 else TOL_BF16)


def test_concurrent_threads_and_streams(la):
    """Calls are pure and reentrant (reference SPEC.md:68): two host threads on their
    own CUDA streams -- plain grid, balanced schedule and in-device split, plus a failing call --
    give bitwise the results of the same calls made serially, and errors stay thread-local."""
    import threading
    from paper_2501_02573_b200 import ops
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    shapes = [(2, 3, 700, 128, 128), (1, sms + 3, 256, 64, 128), (1, 2, 4096, 128, 128)]
    g = torch.Generator(device="cuda").manual_seed(3)
    cases = []
    for (B, H, N, dk, dv) in shapes:
        q = torch.randn(B, H, N, dk, device="cuda", dtype=torch.bfloat16, generator=g)
        k = torch.randn(B, H, N, dk, device="cuda", dtype=torch.bfloat16, generator=g)
        v = torch.randn(B, H, N, dv, device="cuda", dtype=torch.bfloat16, generator=g)
        l2 = ops.log2_gamma([0.9 + 0.09 * (h % 2) for h in range(H)], True, "cuda")
        cases.append((q, k, v, l2))
    serial = [ops.prefill(*c) for c in cases]
    torch.cuda.synchronize()
    results, errors = {}, []

    def worker(tid):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    for i, c in enumerate(cases):
                        results[(tid, rep, i)] = ops.prefill(*c)
                if tid == 1:   # a failing C call on this thread: thread-local status and message
                    from paper_2501_02573_b200 import _lib
                    lib = _lib.load()
                    with pytest.raises(la.ShapeError, match="seqlen"):
                        _lib.check(lib.linattn_prefill(1, 1, 1, 1, 1, None, None, 1, 1, 0, 4, 4, 1, 0, None))
            s.synchronize()
        except Exception as e:   # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for (tid, rep, i), out in results.items():
        assert torch.equal(out, serial[i]), (tid, rep, i)


def _sampled_slices_match(o, q, k, v, gam, picks, tol=TOL_BF16):
    """Sampled (b, h) slices of a full-size output against the seeded f64 blocked oracle."""
    for (bi, h) in picks:
        sl = lambda t: t[bi:bi + 1, h:h + 1].float().cpu().numpy()   # noqa: E731
        ref, _ = orc.seeded_blocked_attn(sl(q), sl(k), sl(v), [gam[h]], True, None, block=64)
        assert orc.max_rel_error(o[bi, h].float().cpu().numpy(), ref[0, 0]) <= tol, (bi, h)


def test_full_size_configs2_configs4_and_balanced(la):
    """Full BASELINE.json sizes the dense oracle cannot take: configs[2] (dk=256/dv=512 clusters),
    configs[4] (N=131072, in-device split) and a 160-unit balanced launch, on sampled slices of
    the f64 blocked oracle; plus the split/no-split agreement and the end state at configs[4]."""
    from paper_2501_02573_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(11)
    for (B, H, N, dk, dv, picks) in [(4, 16, 16384, 256, 512, [(0, 0), (3, 15)]),
                                     (1, 32, 131072, 128, 128, [(0, 0), (0, 31)]),
                                     (5, 32, 8192, 128, 128, [(0, 0), (2, 7), (4, 31)])]:
        q = torch.randn(B, H, N, dk, device="cuda", dtype=torch.bfloat16, generator=g)
        k = torch.randn(B, H, N, dk, device="cuda", dtype=torch.bfloat16, generator=g)
        v = torch.randn(B, H, N, dv, device="cuda", dtype=torch.bfloat16, generator=g)
        gam = [1 - 2.0 ** (-5 - 10 * h / (H - 1)) for h in range(H)]
        l2 = ops.log2_gamma(gam, True, "cuda")
        s_out = torch.empty(B, H, dk, dv, device="cuda")
        o = ops.prefill(q, k, v, l2, s_out=s_out)
        _sampled_slices_match(o, q, k, v, gam, picks)
        if N == 131072:
            one = ops.prefill(q, k, v, l2, seq_split=1)     # single pass, no split
            assert orc.max_rel_error(o.float().cpu().numpy(), one.float().cpu().numpy()) <= TOL_BF16
            ref_s = orc.segment_end_state(k[0, 31].float().cpu().numpy(), v[0, 31].float().cpu().numpy(), gam[31])
            assert orc.max_rel_error(s_out[0, 31].cpu().numpy(), ref_s) <= 5e-3
        del q, k, v, o


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("LINATTN_FUZZ_SEEDS", "48"))))
def test_random_shapes_fuzz(la, seed):
    """Seeded random shapes across every dispatch branch (tensor cores dk in {64,128,256}, FFMA any
    dk/dv, sequence split, balanced schedule, partial dv tiles, ragged N, gamma in {0, 1} and
    near 1), with s_in / s_out, against the seeded f64 blocked oracle."""
    from paper_2501_02573_b200 import ops
    rng = np.random.default_rng(1000 + seed)
    dk = int(rng.choice([8, 24, 64, 128, 256]))
    dv = int(rng.choice([8, 40, 64, 128, 192, 256]))
    B = int(rng.integers(1, 4))
    H = int(rng.choice([1, 2, 3, 5, 40, 100]))
    N = int(rng.choice([1, 17, 64, 100, 333, 1024, 2500]))
    if B * H * N * (dk + dv) > 4e7:             # keep the f64 oracle to a second or two
        N = max(1, int(4e7 // (B * H * (dk + dv))))
    gam = [float(rng.choice([0.0, 1.0, 0.5, 1 - 2.0 ** -6, 1 - 2.0 ** -14])) for _ in range(H)]
    b, c, v = orc.gen_inputs(B, H, N, dk, dv, np.float32, seed)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    s0 = rng.standard_normal((B, H, dk, dv)).astype(np.float32) * 0.05
    ref, ref_s = orc.seeded_blocked_attn(b, c, v, gam, True, s0.astype(np.float64), block=64)
    l2 = ops.log2_gamma(gam, True, "cuda")
    legs = [(torch.bfloat16, "auto", TOL_BF16), (torch.float32, "simt", TOL_F32)]
    if dk <= 128 and dk % 4 == 0 and dv % 4 == 0:
        legs.append((torch.float32, "tf32", TOL_F32))      # the 3xTF32 tensor-core parity mode
    for dt, kernel, tol in legs:
        s_out = torch.full((B, H, dk, dv), float("nan"), device="cuda")
        out = ops.prefill(dev(b, dt), dev(c, dt), dev(v, dt), l2, s_in=dev(s0), s_out=s_out, kernel=kernel)
        assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= tol, (dt, B, H, N, dk, dv)
        assert orc.max_rel_error(s_out.cpu().numpy(), ref_s) <= max(tol, 5e-3), (dt, B, H, N, dk, dv)
        # the row recurrence (b200-recurrent) on the same inputs, where its kernel takes the shape
        ev = 16 // torch.tensor([], dtype=dt).element_size()
        if dk % ev == 0 and dv % ev == 0 and dk <= 256:
            s_rec = torch.empty_like(s_out)
            rec = ops.recurrent(dev(b, dt), dev(c, dt), dev(v, dt), l2, s_in=dev(s0), s_out=s_rec)
            assert orc.max_rel_error(rec.float().cpu().numpy(), ref) <= tol, ("rec", dt, B, H, N, dk, dv)
            assert orc.max_rel_error(s_rec.cpu().numpy(), ref_s) <= max(tol, 1e-5), ("rec", dt, B, H, N, dk, dv)


def test_recurrent_lazy_renormalisation(la):
    """bf16 row recurrence keeps T = S / gamma^t and renormalises before gamma^t underflows:
    small gammas (renormalised every ~20-60 tokens) over a long sequence, with the end state."""
    from paper_2501_02573_b200 import ops
    gam = [0.3, 0.5, 0.7, 0.999]
    b, c, v = (orc.bf16_round(x) for x in orc.gen_inputs(1, 4, 700, 128, 128, np.float32, 23))
    ref, ref_s = orc.seeded_blocked_attn(b, c, v, gam, True, None, block=64)
    l2 = ops.log2_gamma(gam, True, "cuda")
    s_out = torch.empty(1, 4, 128, 128, device="cuda")
    out = ops.recurrent(dev(b, torch.bfloat16), dev(c, torch.bfloat16), dev(v, torch.bfloat16), l2, s_out=s_out)
    assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16
    err_lazy = orc.max_rel_error(s_out.cpu().numpy(), ref_s)          # fp32 state from bf16 inputs
    # the same values as fp32 inputs run the direct form (S <- gamma S + k^T v): the lazy form's
    # state is as accurate (both at the fp32 1e-4 bar; accumulation error of 700 rank-1 updates)
    s32 = torch.empty_like(s_out)
    ops.recurrent(dev(b), dev(c), dev(v), l2, s_out=s32)
    err_direct = orc.max_rel_error(s32.cpu().numpy(), ref_s)
    assert err_lazy <= TOL_F32 and err_direct <= TOL_F32
    assert err_lazy <= 4 * err_direct + 1e-6, (err_lazy, err_direct)


def test_numpy_inputs_concurrent_threads(la):
    """The reference's calling convention (pageable numpy) from two host threads at once: the
    pinned staging buffers are per thread, so results equal the serial ones bitwise."""
    import threading
    rng = np.random.default_rng(9)
    cases = []
    for (B, H, N, d) in [(2, 3, 700, 64), (3, 2, 1300, 128)]:
        b, c, v = (rng.standard_normal((B, H, N, d)).astype(np.float32) for _ in range(3))
        cases.append(la.make_inputs(b, c, v, gamma=[0.9] * H, decay=True))
    methods = ["b200-chunked", "b200-chunked-f32", "b200-recurrent"]
    serial = {(i, m): la.run_method(la.MethodId.parse(m), inp)[0] for i, inp in enumerate(cases) for m in methods}
    got, errors = {}, []

    def worker(order):
        try:
            for rep in range(2):
                for i in order:
                    for m in methods:
                        got[(threading.get_ident(), rep, i, m)] = la.run_method(la.MethodId.parse(m), cases[i])[0]
        except Exception as e:   # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(o,)) for o in ([0, 1], [1, 0])]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for (_, _, i, m), out in got.items():
        assert isinstance(out, np.ndarray) and out.dtype == np.float32
        np.testing.assert_array_equal(out, serial[(i, m)])


@pytest.mark.parametrize("seed", range(16))
def test_decode_fuzz(la, seed):
    """Random decode shapes (few or many states, ragged column slices, odd dv, bf16 / fp32 inputs):
    several steps against the oracle recurrence, state and outputs."""
    from paper_2501_02573_b200 import ops
    rng = np.random.default_rng(500 + seed)
    B, H = int(rng.choice([1, 2, 3, 40])), int(rng.choice([1, 3, 8]))
    dk, dv = int(rng.choice([4, 16, 64, 128, 200])), int(rng.choice([4, 5, 36, 100, 128, 256]))
    gam = [float(rng.choice([0.0, 0.5, 0.95, 1.0])) for _ in range(H)]
    steps = 3
    s0 = rng.standard_normal((B, H, dk, dv)) * 0.1
    q, k, v = (rng.standard_normal((B, H, steps, d)) for d in (dk, dk, dv))
    ref, ref_s = orc.decode_steps(q, k, v, s0, gam)
    st = dev(s0)
    l2 = ops.log2_gamma(gam, True, "cuda")
    outs = [ops.decode_step(dev(q[:, :, i]), dev(k[:, :, i]), dev(v[:, :, i]), st, l2) for i in range(steps)]
    got = torch.stack(outs, 2).cpu().numpy()
    assert orc.max_rel_error(got, ref) <= TOL_F32, (B, H, dk, dv)
    assert orc.max_rel_error(st.cpu().numpy(), ref_s) <= TOL_F32, (B, H, dk, dv)


def test_block_size_honoured_or_rejected(la, golden):
    """BlockParams.block_size (reference kernels.py:47-61): a block of k kernel chunks is k chunks,
    so every positive multiple of the kernel chunk gives the same output (block-size invariance,
    reference test_kernels.py:114-124) with the opcount at the chunk actually used; any other
    value raises UsageError instead of being ignored."""
    from paper_2501_02573_b200 import ops
    from paper_2501_02573_b200.kernels import kernel_chunk
    b, c, v = orc.gen_inputs(2, 3, 333, 64, 64, np.float32, 12)
    gam = [0.0, 0.9, 1.0]
    ref = orc.oracle_attn(orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v), gam, True)
    dev_in = la.make_inputs(*(dev(orc.bf16_round(x), torch.bfloat16) for x in (b, c, v)), gamma=gam, decay=True)
    assert kernel_chunk(la.MethodId.B200_CHUNKED, dev_in) == 64
    outs = {}
    for bs in (64, 128, 256):
        out, opc = la.run_method(la.MethodId.B200_CHUNKED, dev_in, la.BlockParams(block_size=bs))
        outs[bs] = out
        assert opc == ops.chunked_opcount(2, 3, 333, 64, 64, True, 64)
        assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= TOL_BF16
    assert torch.equal(outs[64], outs[128]) and torch.equal(outs[64], outs[256])
    for bad in (1, 32, 48, 0, -64):
        with pytest.raises(la.UsageError):
            la.run_method(la.MethodId.B200_CHUNKED, dev_in, la.BlockParams(block_size=bad))
    f32_in = la.make_inputs(b, c, v, gam, True)                 # host f32: 3xTF32 kernel, chunk 32
    assert kernel_chunk(la.MethodId.B200_CHUNKED_F32, f32_in) == 32
    ref32 = orc.oracle_attn(b, c, v, gam, True)
    prev = None
    for bs in (32, 64, 128):
        out, opc = la.run_method(la.MethodId.B200_CHUNKED_F32, f32_in, la.BlockParams(block_size=bs))
        assert opc == ops.chunked_opcount(2, 3, 333, 64, 64, True, 32)
        assert orc.max_rel_error(out, ref32) <= TOL_F32
        if prev is not None:
            np.testing.assert_array_equal(out, prev)
        prev = out
    with pytest.raises(la.UsageError):
        la.run_method(la.MethodId.B200_CHUNKED_F32, f32_in, la.BlockParams(block_size=16))
    # the row recurrence has no chunk: any block size is accepted
    la.run_method(la.MethodId.B200_RECURRENT, f32_in, la.BlockParams(block_size=7))
