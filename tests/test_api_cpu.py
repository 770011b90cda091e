"""Host-side logic that runs without a GPU: the entry contract, dispatch, the ABI surface."""

import os
import re
import subprocess

import numpy as np
import pytest
import torch

import paper_2501_02573_b200 as la
from paper_2501_02573_b200 import _lib, ops
from paper_2501_02573_b200.sp import segment_bounds

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "linattn_b200.h")


# --- entry contract (reference tensor.py:97-144, test_tensor.py) ---------------

def test_make_inputs_broadcasts_and_defaults():
    inp = la.make_inputs([[2.0], [3.0]], [[1.0], [4.0]], [[5.0], [6.0]])
    assert inp.b.shape == (1, 1, 2, 1) and inp.b.dtype == np.float64
    assert inp.gamma == [1.0] and inp.decay is False
    inp = la.make_inputs(np.ones((3, 2), np.float32), np.ones((3, 2), np.float32), np.ones((3, 4), np.float32),
                         gamma=0.5, decay=True)
    assert inp.v.dtype == np.float32 and inp.gamma == [0.5]
    ints = la.make_inputs(np.ones((2, 1), np.int32), np.ones((2, 1), np.int32), np.ones((2, 1), np.int32))
    assert ints.b.dtype == np.float64  # upcast like the reference (tensor.py:31-32)


def test_validate_names_axis_and_flat_index():
    rng = np.random.default_rng(17)
    inp = la.AttnInputs(b=rng.standard_normal((1, 2, 8, 4)), c=rng.standard_normal((1, 2, 8, 5)),
                        v=rng.standard_normal((1, 2, 8, 16)), gamma=[0.9, 0.9])
    with pytest.raises(la.ShapeError, match="rank"):
        la.validate_inputs(inp)
    v = np.ones((1, 1, 3, 2))
    v[0, 0, 2, 1] = np.nan
    with pytest.raises(la.DataError, match="flat index 5"):
        la.validate_inputs(la.AttnInputs(b=np.ones((1, 1, 3, 2)), c=np.ones((1, 1, 3, 2)), v=v, gamma=[1.0]))
    with pytest.raises(la.ParameterError):
        la.make_inputs(np.ones((2, 1)), np.ones((2, 1)), np.ones((2, 1)), gamma=[1.2])
    with pytest.raises(la.ShapeError):
        la.make_inputs(np.ones((0, 1)), np.ones((0, 1)), np.ones((0, 1)))


def test_validate_device_tensor_types_on_cpu_torch():
    # torch tensors take the device path; bf16 is an accepted dtype there
    t = torch.ones(1, 1, 4, 2, dtype=torch.bfloat16)
    inp = la.make_inputs(t, t, torch.ones(1, 1, 4, 3, dtype=torch.bfloat16), gamma=0.9, decay=True)
    assert inp.on_device and inp.v.dtype == torch.bfloat16
    bad = torch.ones(1, 1, 4, 2)
    bad[0, 0, 1, 1] = float("inf")
    with pytest.raises(la.DataError, match="flat index 3"):
        la.make_inputs(bad, bad, bad)


# --- methods and dispatch (reference kernels.py:25-44, dispatch.py) ---------------

def test_method_parse_and_reference_names():
    assert la.MethodId.parse("b200-chunked") is la.MethodId.B200_CHUNKED
    with pytest.raises(la.UsageError, match="CPU route of the reference"):
        la.MethodId.parse("two-level-block")
    with pytest.raises(la.UsageError, match="unknown method"):
        la.MethodId.parse("nosuch")


def test_run_method_rejects_auto():
    inp = la.make_inputs(np.ones((4, 2)), np.ones((4, 2)), np.ones((4, 2)))
    with pytest.raises(la.UsageError):
        la.run_method(la.MethodId.AUTO, inp)


def test_default_policy_resolves_on_precision():
    pol = la.default_policy()
    assert pol.resolve(8, 8192, True, "bf16")[0] is la.MethodId.B200_CHUNKED
    assert pol.resolve(1, 100, False, "f32")[0] is la.MethodId.B200_CHUNKED_F32
    inp = la.make_inputs(np.ones((4, 2)), np.ones((4, 2)), np.ones((4, 2)))
    assert la.explain(inp)[0] is la.MethodId.B200_CHUNKED_F32


def test_policy_file_grammar(tmp_path):
    text = """
    # reference 6-field lines plus an optional dtype field
    1,1,*,128,binary,b200-recurrent
    *,*,*,*,*,b200-chunked,bf16
    """
    pol = la.parse_policy(text)
    assert pol.resolve(1, 100, False, "f32")[0] is la.MethodId.B200_RECURRENT
    assert pol.resolve(4, 100, True, "bf16")[0] is la.MethodId.B200_CHUNKED
    assert pol.resolve(4, 100, True, "f32")[0] is pol.default
    p = tmp_path / "policy.txt"
    p.write_text(text)
    assert la.load_policy(str(p)).resolve(1, 5, False, "f32")[0] is la.MethodId.B200_RECURRENT
    for bad in ("1,1,binary,b200-chunked", "1,1,*,*,binary,nosuch", "1,1,*,*,binary,auto",
                "x,1,*,*,binary,b200-chunked", "*,*,*,*,*,b200-chunked,fp8"):
        with pytest.raises(la.UsageError):
            la.parse_policy(bad)


def test_no_cpu_fallback_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    inp = la.make_inputs(np.ones((4, 2)), np.ones((4, 2)), np.ones((4, 2)))
    with pytest.raises((la.LinAttnError, RuntimeError, AssertionError)):
        la.run_method(la.MethodId.B200_CHUNKED_F32, inp)


# --- analytic accounting ---------------------------------------------------------

def test_opcount_matches_reference_formula():
    # two-level-block decay opcount per block: L^2 (r+d+1) + 2Lr + 2Lrd + rd (kernels.py:158-159)
    n, r, d, C = 130, 4, 6, 64
    want = 0
    for L in (64, 64, 2):
        want += L * L * (r + d + 1) + 2 * L * r + 2 * L * r * d + r * d
    assert ops.chunked_opcount(2, 3, n, r, d, True, C) == 6 * want
    assert ops.bytes_per_token_head(128, 128) == 1024


def test_log2_gamma_conventions():
    l2 = ops.log2_gamma([0.0, 0.5, 1.0], True).numpy()
    assert np.isneginf(l2[0]) and l2[1] == -1.0 and l2[2] == 0.0
    assert np.all(ops.log2_gamma([0.0, 0.5], False).numpy() == 0.0)
    # f64-derived log2 keeps gamma^n accurate at n = 131072
    g = 1 - 4.6e-6
    approx = 2.0 ** (131072 * np.float64(ops.log2_gamma([g], True).numpy()[0]))
    assert abs(approx / g ** 131072 - 1) < 1e-5


def test_segment_bounds():
    assert segment_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert segment_bounds(131072, 8)[-1] == (114688, 131072)


# --- the C ABI surface -------------------------------------------------------------

def _declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"LINATTN_API\s+[\w\s\*]+?\b(linattn_\w+)\s*\(", text)))


def test_header_declares_what_the_binding_uses():
    assert _declared_symbols() == sorted(_lib.EXPORTED)


@pytest.mark.skipif(not os.path.exists(_lib.LIB_PATH), reason="library not built")
def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (linattn_\w+)", out))
    assert set(_declared_symbols()) <= exported
    lib = _lib.load()
    assert lib.linattn_abi_version() == _lib.ABI_VERSION


@pytest.mark.skipif(not os.path.exists(_lib.LIB_PATH), reason="library not built")
def test_host_validation_errors_without_gpu():
    # shape/parameter checks happen on the host before any launch, so they work without a GPU
    lib = _lib.load()
    with pytest.raises(la.ShapeError, match="seqlen"):
        _lib.check(lib.linattn_prefill(1, 1, 1, 1, 1, None, None, 1, 1, 0, 4, 4, 1, 0, None))
    with pytest.raises(la.UsageError, match="dtype"):
        _lib.check(lib.linattn_prefill(1, 1, 1, 1, 1, None, None, 1, 1, 8, 4, 4, 7, 0, None))
    with pytest.raises(la.UsageError, match="tensor-core"):
        _lib.check(lib.linattn_prefill(1, 1, 1, 1, 1, None, None, 1, 1, 8, 4, 4, 0, 1, None))
    with pytest.raises(la.UsageError, match="65535"):
        _lib.check(lib.linattn_prefill(1, 1, 1, 1, 1, None, None, 256, 257, 8, 4, 4, 1, 0, None))
    with pytest.raises(la.ParameterError):
        import ctypes
        lens = (ctypes.c_int64 * 2)(1, 2)
        _lib.check(lib.linattn_prefix_combine(1, 1, lens, 2, 5, 1, 1, 1, 4, 4, None))


def test_bench_summarize_matches_reference_arithmetic():
    """summarize() keeps the reference contract (reference tests/test_bench.py:20-36)."""
    import math
    import numpy as np
    from paper_2501_02573_b200 import UsageError, summarize
    mean, std = summarize([3, 1, 2, 9, 2], drop_extremes=True)
    assert mean == pytest.approx(7 / 3) and std == pytest.approx(np.std([3, 2, 2], ddof=1))
    assert summarize([2, 2, 2]) == (2, 0)
    mean, std = summarize([1.0, 2.0, 3.0, 4.0])
    assert mean == 2.5 and std == pytest.approx(math.sqrt(5 / 3))
    with pytest.raises(UsageError):
        summarize([1, 2], drop_extremes=True)


def test_bench_gen_inputs_bitwise_reference_stream():
    """gen_inputs draws the reference's PCG64 stream (bench.py:77-84) == the oracle's."""
    import numpy as np
    from oracle import linattn_oracle as orc
    from paper_2501_02573_b200 import gen_inputs
    a = gen_inputs(2, 3, 16, 4, 5, np.float32, seed=9, decay=True, gamma=0.7)
    b, c, v = orc.gen_inputs(2, 3, 16, 4, 5, np.float32, 9)
    assert np.array_equal(a.b, b) and np.array_equal(a.c, c) and np.array_equal(a.v, v)
    assert a.gamma == [0.7] * 3 and a.decay
    assert not np.array_equal(gen_inputs(2, 3, 16, 4, 5, np.float32, seed=10).b, a.b)


def test_bench_render_and_usage_errors():
    from paper_2501_02573_b200 import BenchConfig, MethodId, UsageError, render_report, run_bench
    from paper_2501_02573_b200.bench import BenchReport, BenchRow
    row = BenchRow(MethodId.B200_CHUNKED, 1, 2, 64, 8, 8, "decay", 0.9, "bf16", 1e-4, 1e-6, 123, "ok",
                   100.0, 0.5, 1.0)
    oom = BenchRow(MethodId.B200_CHUNKED_F32, 1, 2, 64, 8, 8, "decay", 0.9, "f32", None, None, None, "OOM")
    rep = BenchReport(rows=[row, oom], meta={"seed": 0})
    csv = render_report(rep, "csv").splitlines()
    assert csv[0].startswith("method,batch,heads,seqlen") and csv[0].endswith("gbps,frac_hbm,tflops_c64")
    assert csv[1].startswith("b200-chunked,1,2,64,8,8,decay,0.9,bf16,0.0001,") and csv[2].endswith("OOM,,,")
    md = render_report(rep, "markdown")
    assert "| b200-chunked |" in md and "OOM" in md and "50% HBM" in md
    with pytest.raises(UsageError):
        render_report(rep, "xml")
    with pytest.raises(UsageError):
        run_bench(BenchConfig(methods=[MethodId.AUTO], grid=[(1, 1, 8, 2, 2)]))
    with pytest.raises(UsageError):
        run_bench(BenchConfig(methods=[MethodId.B200_CHUNKED], grid=[]))


def test_release_staging_buffers_is_safe_without_gpu():
    from paper_2501_02573_b200 import release_staging_buffers
    release_staging_buffers()
    release_staging_buffers()
