"""Parity at the operating points bench.py actually times, plus the front-door contract on device.

* configs[3] decode: bf16 q/k/v, B=256, H=32, d=128, 1024 steps, the un-split grid (8192 states
  fill the SMs, one CTA per state) -- sampled states and outputs against the f64 row recurrence
  (reference _row_based_slice, kernels.py:93-106), and the CUDA-graph replay the bench uses
  bit-identical to eager launches;
* a bf16 multi-step decode fuzz over split and un-split grids;
* configs[4] (B=1, H=32, N=131072, d=128): the last 2048 tokens of EVERY head and every end state
  against an f64 reference seeded with the exact f64 prefix state;
* ops wrappers reject mismatched shapes/dtypes before calling into C;
* the fused device finiteness scan names the first non-finite flat index like the reference
  check_finite (tensor.py:20-25) and is not repeated for unmodified tensors.
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


def _gammas(h):
    return [1.0 - 2.0 ** (-5 - 10 * i / max(1, h - 1)) for i in range(h)]


def test_configs3_decode_bf16_1024_steps(ops):
    B, H, d, T = 256, 32, 128, 1024
    g = torch.Generator(device="cuda").manual_seed(31)
    gam = _gammas(H)
    gam[3] = 0.0                      # gamma = 0 and 1 heads on the benched grid too
    gam[4] = 1.0
    l2 = ops.log2_gamma(gam, True, "cuda")
    # per-step inputs [T, B, H, d] bf16 (2 GiB each), scaled like the bench
    q = (torch.randn(T, B, H, d, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    k = (torch.randn(T, B, H, d, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    v = (torch.randn(T, B, H, d, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    state = torch.zeros(B, H, d, d, device="cuda")
    out = torch.empty(T, B, H, d, device="cuda", dtype=torch.bfloat16)
    for t in range(T):
        ops.decode_step(q[t], k[t], v[t], state, l2, out=out[t])
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    picks = [(int(b), int(h)) for b, h in zip(rng.integers(0, B, 14), rng.integers(0, H, 14))]
    picks += [(0, 3), (B - 1, 4)]
    for b, h in picks:
        qq, kk, vv = (x[:, b, h].double().cpu().numpy()[None, None] for x in (q, k, v))
        ref, ref_s = orc.decode_steps(qq, kk, vv, np.zeros((1, 1, d, d)), [gam[h]])
        got = out[:, b, h].float().cpu().numpy()
        assert orc.max_rel_error(got, ref[0, 0]) <= TOL_BF16, (b, h)
        assert orc.max_rel_error(state[b, h].cpu().numpy(), ref_s[0, 0]) <= TOL_F32, (b, h)


def test_configs3_decode_graph_replay_matches_eager(ops):
    """bench.py times 64-step CUDA graphs of decode_step on one set of inputs: the replay must be
    bit-identical to eager launches on the same inputs."""
    B, H, d = 256, 32, 128
    g = torch.Generator(device="cuda").manual_seed(7)
    qd, kd, vd = ((torch.randn(B, H, d, device="cuda", generator=g) * 0.1).to(torch.bfloat16) for _ in range(3))
    l2 = ops.log2_gamma(_gammas(H), True, "cuda")
    s_eager = torch.zeros(B, H, d, d, device="cuda")
    s_graph = torch.zeros_like(s_eager)
    o_eager = torch.empty_like(vd)
    o_graph = torch.empty_like(vd)
    for _ in range(64):
        ops.decode_step(qd, kd, vd, s_eager, l2, out=o_eager)
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            for _ in range(64):
                ops.decode_step(qd, kd, vd, s_graph, l2, out=o_graph)
    torch.cuda.current_stream().wait_stream(side)
    s_graph.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(s_graph, s_eager)
    assert torch.equal(o_graph, o_eager)


@pytest.mark.parametrize("seed", range(12))
def test_decode_fuzz_bf16(ops, seed):
    """bf16 q/k/v, many steps, split (few states) and un-split (many states) grids."""
    rng = np.random.default_rng(900 + seed)
    B, H = int(rng.choice([1, 2, 64, 300])), int(rng.choice([1, 4, 32]))
    dk, dv = int(rng.choice([8, 64, 128, 256])), int(rng.choice([8, 64, 128, 136, 512]))
    steps = int(rng.choice([17, 64]))
    gam = [float(rng.choice([0.0, 0.5, 0.97, 1 - 2.0 ** -12, 1.0])) for _ in range(H)]
    q, k, v = (orc.bf16_round(rng.standard_normal((B, H, steps, dd)) * 0.2) for dd in (dk, dk, dv))
    s0 = rng.standard_normal((B, H, dk, dv)) * 0.1
    picks = [(int(b), int(h)) for b, h in zip(rng.integers(0, B, 6), rng.integers(0, H, 6))]
    st = torch.from_numpy(s0).to("cuda", torch.float32)
    l2 = ops.log2_gamma(gam, True, "cuda")
    qd, kd, vd = (torch.from_numpy(x).to("cuda", torch.bfloat16) for x in (q, k, v))
    outs = [ops.decode_step(qd[:, :, i].contiguous(), kd[:, :, i].contiguous(), vd[:, :, i].contiguous(), st, l2)
            for i in range(steps)]
    got = torch.stack(outs, 2).float().cpu().numpy()
    s_got = st.cpu().numpy()
    for b, h in picks:
        ref, ref_s = orc.decode_steps(q[b:b + 1, h:h + 1], k[b:b + 1, h:h + 1], v[b:b + 1, h:h + 1],
                                      s0[b:b + 1, h:h + 1], [gam[h]])
        assert orc.max_rel_error(got[b, h], ref[0, 0]) <= TOL_BF16, (B, H, dk, dv, b, h)
        assert orc.max_rel_error(s_got[b, h], ref_s[0, 0]) <= TOL_F32, (B, H, dk, dv, b, h)


def test_configs4_every_head(ops):
    """configs[4] as benched on one GPU (in-device sequence split): the last 2048 tokens of all 32
    heads and all 32 end states against f64 references seeded with the exact f64 prefix state."""
    B, H, N, d, T = 1, 32, 131072, 128, 2048
    g = torch.Generator(device="cuda").manual_seed(17)
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16, generator=g)
    k = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16, generator=g)
    v = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16, generator=g)
    gam = _gammas(H)
    l2 = ops.log2_gamma(gam, True, "cuda")
    assert ops.seq_plan(B, H, N, d, d)[1] > 1
    s_out = torch.empty(B, H, d, d, device="cuda")
    o = ops.prefill(q, k, v, l2, s_out=s_out)
    for h in range(H):
        kk = k[0, h].double().cpu().numpy()
        vv = v[0, h].double().cpu().numpy()
        lg = np.log(gam[h])
        w = np.exp((N - T - 1 - np.arange(N - T)) * lg)                 # f64 gamma^(L-1-t)
        s_pre = (kk[:N - T] * w[:, None]).T @ vv[:N - T]
        qq = q[0, h, N - T:].double().cpu().numpy()
        ref, s_end = orc.seeded_blocked_attn(qq[None, None], kk[None, None, N - T:], vv[None, None, N - T:],
                                             [gam[h]], True, s_pre[None, None], block=64)
        assert orc.max_rel_error(o[0, h, N - T:].float().cpu().numpy(), ref[0, 0]) <= TOL_BF16, h
        assert orc.max_rel_error(s_out[0, h].cpu().numpy(), s_end[0, 0]) <= 5e-3, h


def test_ops_reject_mismatched_shapes(ops):
    from paper_2501_02573_b200.errors import ShapeError, UsageError
    q = torch.zeros(2, 3, 128, device="cuda")
    st = torch.zeros(2, 3, 128, 64, device="cuda")
    l2 = ops.log2_gamma([0.9] * 3, True, "cuda")
    with pytest.raises(ShapeError):
        ops.decode_step(q, torch.zeros(2, 3, 64, device="cuda"), torch.zeros(2, 3, 64, device="cuda"), st, l2)
    with pytest.raises(ShapeError):
        ops.decode_step(q, q, torch.zeros(2, 2, 64, device="cuda"), st, l2)
    with pytest.raises(UsageError):
        ops.decode_step(q, q.bfloat16(), torch.zeros(2, 3, 64, device="cuda"), st, l2)
    with pytest.raises(ShapeError):
        ops.decode_step(q, q, torch.zeros(2, 3, 64, device="cuda"), st, l2[:2])
    x = torch.zeros(1, 3, 100, 64, device="cuda")
    with pytest.raises(ShapeError):
        ops.recurrent(x, x, torch.zeros(1, 3, 99, 64, device="cuda"), l2)
    with pytest.raises(ShapeError):
        ops.recurrent(x, x, x, l2, s_out=torch.zeros(1, 3, 64, 32, device="cuda"))
    with pytest.raises(ShapeError):
        ops.state_pass(x, torch.zeros(1, 2, 100, 64, device="cuda"), l2)
    with pytest.raises(ShapeError):
        ops.prefill(x, x, x, l2, out=torch.zeros(1, 3, 100, 32, device="cuda"))
    with pytest.raises(UsageError):
        ops.prefill(x, x, x.bfloat16(), l2)


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_device_finiteness_scan(ops, dt):
    """validate_inputs on CUDA tensors: one fused scan names the first non-finite flat index like
    the reference check_finite (tensor.py:20-25), incl. 16-byte unaligned views; decode on the
    same inputs raises the same DataError through its deferred (output-first) check."""
    import paper_2501_02573_b200 as la
    from paper_2501_02573_b200.errors import DataError
    n = 1 << 20
    for name, which, idx, offset in [("B", 0, 0, 0), ("C", 1, n - 1, 0), ("V", 2, 12345, 3), ("C", 1, 7, 1)]:
        base = [torch.randn(n + offset, device="cuda").to(dt) for _ in range(3)]
        views = [x[offset:].view(1, 1, n // 64, 64) for x in base]   # offset: 16-byte unaligned views
        views[which].view(-1)[idx] = float("inf") if idx % 2 else float("nan")
        inp = la.make_inputs(*views, gamma=0.9, decay=True)
        with pytest.raises(DataError, match=f"{name} has a non-finite entry at flat index {idx}$"):
            la.validate_inputs(inp)
        inp = la.make_inputs(*views, gamma=0.9, decay=True)
        with pytest.raises(DataError, match=f"{name} has a non-finite entry at flat index {idx}$"):
            la.decode(inp)
    # first offending tensor in B, C, V order, smallest index within it
    xs = [torch.randn(4, 2, 50, 16, device="cuda").to(dt) for _ in range(3)]
    xs[2].view(-1)[3] = float("nan")
    xs[1].view(-1)[900] = float("nan")
    xs[1].view(-1)[77] = float("inf")
    with pytest.raises(DataError, match="C has a non-finite entry at flat index 77$"):
        la.decode(la.make_inputs(*xs, gamma=0.5, decay=True))


@pytest.mark.parametrize("gamma", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("which", [0, 1, 2])
def test_nonfinite_input_always_reaches_the_output(ops, gamma, which):
    """The deferred check relies on every NaN/Inf input element reaching some output (a masked
    product is NaN, not 0): one bad element anywhere, each method, gamma in {0, 0.5, 1}."""
    import paper_2501_02573_b200 as la
    from paper_2501_02573_b200.errors import DataError
    rng = np.random.default_rng(which)
    for method, dt, (dk, dv) in [("b200-chunked", torch.bfloat16, (128, 128)), ("b200-chunked", torch.bfloat16, (256, 512)),
                                 ("b200-chunked", torch.bfloat16, (24, 40)), ("b200-chunked-f32", torch.float32, (64, 64)),
                                 ("b200-chunked-f32", torch.float32, (6, 10)), ("b200-recurrent", torch.float32, (64, 64)),
                                 ("b200-seqpar", torch.bfloat16, (128, 128))]:
        N = 300
        xs = [torch.randn(2, 3, N, d, device="cuda").to(dt) for d in (dk, dk, dv)]
        pos = int(rng.integers(0, xs[which].numel()))
        xs[which].view(-1)[pos] = float("nan") if pos % 2 else float("-inf")
        with pytest.raises(DataError, match=f"{'BCV'[which]} has a non-finite entry at flat index {pos}$"):
            la.decode(la.make_inputs(*xs, gamma=gamma, decay=True), method=method)


def test_validation_runs_once_until_modified(ops):
    """make_inputs -> decode on CUDA tensors: no input scan at all when the output is finite (the
    bf16 tensor-core prefill checks its outputs in its epilogue: one launch; other kernels add one
    output scan); the next decode of the same unmodified inputs only runs the prefill; an
    in-place write makes the check run again."""
    import paper_2501_02573_b200 as la
    from paper_2501_02573_b200 import _lib
    from paper_2501_02573_b200.errors import DataError
    xs = [torch.randn(2, 4, 256, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
    inp = la.make_inputs(*xs, gamma=0.9, decay=True)
    torch.cuda.synchronize()
    n0 = _lib.launch_count()
    la.decode(inp)
    torch.cuda.synchronize()
    assert _lib.launch_count() - n0 == 1                   # prefill with the fused output check
    f32 = la.make_inputs(*(x.float() for x in xs), gamma=0.9, decay=True)
    n0 = _lib.launch_count()
    la.decode(f32)
    torch.cuda.synchronize()
    assert _lib.launch_count() - n0 == 2                   # 3xTF32 prefill + one output scan
    n0 = _lib.launch_count()
    la.decode(inp)
    torch.cuda.synchronize()
    assert _lib.launch_count() - n0 == 1                   # already established: prefill only
    xs[1][0, 0, 5, 3] = float("nan")                       # in-place write bumps the tensor version
    with pytest.raises(DataError, match="C has a non-finite entry at flat index 323$"):
        la.decode(inp)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_tensors_on_non_current_device(ops):
    """Tensors on cuda:1 while cuda:0 is current launch on cuda:1."""
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 1)
    rng = np.random.default_rng(2)
    b, c, v = (orc.bf16_round(rng.standard_normal((1, 2, 300, 64))) for _ in range(3))
    q, k, vv = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in (b, c, v))
    l2 = ops.log2_gamma([0.9, 1.0], True, dev)
    out = ops.prefill(q, k, vv, l2)
    assert out.device == dev
    assert orc.max_rel_error(out.float().cpu().numpy(), orc.oracle_attn(b, c, v, [0.9, 1.0], True)) <= TOL_BF16


def test_device_oom_is_resource_error(ops):
    """Device memory exhaustion surfaces as the reference's ResourceError (errors.py:25), and the
    package run_bench turns it into an OOM row (reference bench.py:116-117) and carries on."""
    import paper_2501_02573_b200 as la
    from paper_2501_02573_b200.bench import BenchConfig, run_bench
    free, total = torch.cuda.mem_get_info()
    torch.cuda.empty_cache()
    frac = min(1.0, (torch.cuda.memory_allocated() + (64 << 20)) / total)   # ~64 MiB of headroom
    torch.cuda.set_per_process_memory_fraction(frac)
    try:
        big = la.make_inputs(*(torch.ones(1, 8, 65536, 128) for _ in range(3)), gamma=[0.9] * 8)
        with pytest.raises(la.ResourceError):
            la.run_method(la.MethodId.B200_CHUNKED, big)
        cfg = BenchConfig(methods=[la.MethodId.B200_CHUNKED], grid=[(1, 8, 65536, 128, 128), (1, 2, 256, 64, 64)],
                          repeats=1, warmup=0)
        rows = {r.seqlen: r for r in run_bench(cfg).rows}
        assert rows[65536].status == "OOM" and rows[256].status == "ok"
    finally:
        torch.cuda.set_per_process_memory_fraction(1.0)
        torch.cuda.empty_cache()
