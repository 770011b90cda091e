"""Device-level operators over torch CUDA tensors (thin wrappers of the C ABI).

These are the hot-path entry points used by ``run_method``, the decode API,
the sequence-parallel driver and the benchmark.  They validate only what the
C side cannot see (device, contiguity, dtype agreement); shape checks happen
in C (include/linattn_b200.h) and surface as the reference exception classes.
Every call is asynchronous on torch's current CUDA stream.
"""

from __future__ import annotations

import ctypes
import functools

import numpy as np
import torch

from . import _lib
from .errors import LinAttnError, ShapeError, UsageError

_DTYPES = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16}
_KERNELS = {"auto": _lib.KERNEL_AUTO, "tc": _lib.KERNEL_TC, "simt": _lib.KERNEL_SIMT, "tf32": _lib.KERNEL_TF32}


def _require_cuda(*ts):
    """Every given tensor is a contiguous CUDA tensor, all on one device."""
    if not torch.cuda.is_available():
        raise LinAttnError("no CUDA device: the B200 path has no CPU fallback")
    dev = None
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise UsageError("tensor is not on a CUDA device")
        if not t.is_contiguous():
            raise UsageError("tensor must be contiguous")
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise UsageError(f"tensors on different devices: {dev} and {t.device}")


def _on_tensor_device(fn):
    """Run ``fn`` with its first tensor argument's CUDA device current.

    The library reads cudaGetDevice() (SM count, workspace pool, kernel attributes) and every
    launch goes to torch's current stream of the current device, so a call with tensors on
    cuda:1 while cuda:0 is current must switch devices first.
    """
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        t0 = next((a for a in args if isinstance(a, torch.Tensor)), None)
        if t0 is None or not t0.is_cuda or t0.device == torch.device("cuda", torch.cuda.current_device()):
            return fn(*args, **kwargs)
        with torch.cuda.device(t0.device):
            return fn(*args, **kwargs)
    return wrapper


def _check_kv(k, v, ndim: int = 4):
    """k [..., dk] and v [..., dv] agree on every leading axis and share a dtype."""
    if k.dim() != ndim or v.dim() != ndim or tuple(v.shape[:-1]) != tuple(k.shape[:-1]):
        raise ShapeError(f"expected k [..., dk] and v [..., dv] with {ndim} dims and equal leading axes; "
                         f"got {tuple(k.shape)}, {tuple(v.shape)}")
    if k.dtype != v.dtype:
        raise UsageError(f"dtype mismatch: k={k.dtype} v={v.dtype}")


def _check_qkv(q, k, v, ndim: int = 4):
    """q, k [..., dk] of equal shape and v [..., dv] agreeing on the leading axes; one dtype."""
    _check_kv(k, v, ndim)
    if tuple(q.shape) != tuple(k.shape):
        raise ShapeError(f"q and k must have the same shape; got {tuple(q.shape)}, {tuple(k.shape)}")
    if q.dtype != k.dtype:
        raise UsageError(f"dtype mismatch: q={q.dtype} k={k.dtype} v={v.dtype}")


def _check_state(st, shape, what="state"):
    if st is not None and (st.dtype != torch.float32 or tuple(st.shape) != tuple(shape)):
        raise ShapeError(f"{what} must be float32 {list(shape)}, got {st.dtype} {tuple(st.shape)}")


def _check_log2g(log2g, heads: int):
    if log2g.dtype != torch.float32 or log2g.dim() != 1 or log2g.shape[0] < heads:
        raise ShapeError(f"log2g must be float32 [H] with H >= {heads}, got {log2g.dtype} {tuple(log2g.shape)}")


def _dtype_code(t: torch.Tensor) -> int:
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise UsageError(f"unsupported device dtype {t.dtype} (expected float32 or bfloat16)")


def _ptr(t):
    return None if t is None else ctypes_ptr(t)


def ctypes_ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def log2_gamma(gammas, decay: bool = True, device=None) -> torch.Tensor:
    """fp32 log2(gamma) per head, computed in f64 ("decay numerics").

    -inf for gamma == 0 (so gamma^n == 0 for n > 0 while gamma^0 stays 1), 0 for
    gamma == 1 and for the binary mask (decay=False; the reference ignores gamma
    then, e.g. kernels.py:101).
    """
    g = np.asarray(gammas, dtype=np.float64).reshape(-1)
    if decay:
        with np.errstate(divide="ignore"):
            l2 = np.log2(g)
    else:
        l2 = np.zeros_like(g)
    t = torch.from_numpy(l2.astype(np.float32))
    return t.to(device) if device is not None else t


_L2G_CACHE: dict = {}


def log2_gamma_cached(gammas, decay: bool, device) -> torch.Tensor:
    """log2_gamma on ``device``, cached per (gammas, decay, device) for the library's own calls
    (saves a pageable host-to-device copy per call); callers must not modify the result."""
    dev = torch.device(device)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (tuple(float(g) for g in gammas), bool(decay), dev)
    t = _L2G_CACHE.get(key)
    if t is None:
        if len(_L2G_CACHE) > 256:
            _L2G_CACHE.clear()
        t = _L2G_CACHE[key] = log2_gamma(gammas, decay, dev)
    return t


_MAX_GRID_Y = 65535   # the sequence kernels put batch*heads on grid.y


def _batch_chunks(B: int, H: int):
    """Contiguous batch ranges with at most 65535 (batch, head) units each (one launch each)."""
    if B * H <= _MAX_GRID_Y or H > _MAX_GRID_Y:
        return [(0, B)]
    step = _MAX_GRID_Y // H
    return [(b0, min(B, b0 + step)) for b0 in range(0, B, step)]


@_on_tensor_device
def prefill(q, k, v, log2g, *, s_in=None, s_out=None, out=None, kernel: str = "auto",
            seq_split: int | None = None, nonfinite=None):
    """O = (Q K^T (.) M_gamma) V on device; optional initial/end state (fp32).

    ``seq_split``: None lets the library split the sequence across SMs when batch x head
    leaves them idle (``seq_plan``); 1 forces a single pass; P > 1 forces P segments
    (two-phase: segment-local state pass, then every segment seeded in parallel).
    ``nonfinite``: optional int64 [1] CUDA tensor holding INT64_MAX; lowered if the output holds a
    NaN/Inf (fused into the bf16 tensor-core kernel's epilogue, else one scan of the output).
    """
    if nonfinite is not None and seq_split is not None:
        out = prefill(q, k, v, log2g, s_in=s_in, s_out=s_out, out=out, kernel=kernel, seq_split=seq_split)
        _lib.check(_lib.load().linattn_nonfinite_index(out.data_ptr(), out.numel(), _dtype_code(out),
                                                      nonfinite.data_ptr(), _stream()))
        return out
    if seq_split is not None and seq_split > 1:
        n = q.shape[2]
        seg = -(-n // seq_split)
        seg = -(-seg // 64) * 64 if seg < n else n
        nseg = -(-n // seg)
        incl = None
        if nseg > 1:
            loc = state_pass_segmented(k, v, log2g, seg, m=1, nseg=nseg - 1, kernel=kernel)
            incl = segment_prefix(loc, (seg, 1), seg, nseg - 1, log2g, n)
        return prefill_segmented(q, k, v, log2g, seg, loc=incl, loc_geom=(seg, 1), inclusive=True, s_in=s_in,
                                 s_out=s_out, out=out, kernel=kernel)
    if seq_split == 1:
        return prefill_segmented(q, k, v, log2g, q.shape[2], s_in=s_in, s_out=s_out, out=out, kernel=kernel)
    _require_cuda(q, k, v, log2g, s_in, s_out, out)
    _check_qkv(q, k, v)
    B, H, N, dk = q.shape
    dv = v.shape[3]
    _check_log2g(log2g, H)
    if out is None:
        out = torch.empty_like(v)
    if tuple(out.shape) != tuple(v.shape) or out.dtype != v.dtype:
        raise ShapeError(f"out must be {v.dtype} {tuple(v.shape)}, got {out.dtype} {tuple(out.shape)}")
    for st in (s_in, s_out):
        _check_state(st, (B, H, dk, dv))
    lib = _lib.load()
    for b0, b1 in _batch_chunks(B, H):   # more than 65535 (batch, head) units: one launch per chunk
        sl = (lambda t: None if t is None else t[b0:b1])   # noqa: E731
        args = (q[b0:b1].data_ptr(), k[b0:b1].data_ptr(), v[b0:b1].data_ptr(), out[b0:b1].data_ptr(),
                log2g.data_ptr(), _ptr(sl(s_in)), _ptr(sl(s_out)), b1 - b0, H, N, dk, dv, _dtype_code(q),
                _KERNELS[kernel])
        if nonfinite is None:
            _lib.check(lib.linattn_prefill(*args, _stream()))
        else:
            _lib.check(lib.linattn_prefill_checked(*args, nonfinite.data_ptr(), _stream()))
    return out


@_on_tensor_device
def state_pass(k, v, log2g, *, s_out=None, kernel: str = "auto"):
    """End state sum_t gamma^(N-1-t) k_t^T v_t of each (b, h) segment (fp32)."""
    _require_cuda(k, v, log2g, s_out)
    _check_kv(k, v)
    B, H, N, dk = k.shape
    dv = v.shape[3]
    _check_log2g(log2g, H)
    _check_state(s_out, (B, H, dk, dv), "s_out")
    if s_out is None:
        s_out = torch.empty((B, H, dk, dv), dtype=torch.float32, device=k.device)
    lib = _lib.load()
    for b0, b1 in _batch_chunks(B, H):
        _lib.check(lib.linattn_state_pass(k[b0:b1].data_ptr(), v[b0:b1].data_ptr(), s_out[b0:b1].data_ptr(),
                                          log2g.data_ptr(), b1 - b0, H, N, dk, dv, _dtype_code(k),
                                          _KERNELS[kernel], _stream()))
    return s_out


def seq_plan(B: int, H: int, N: int, dk: int, dv: int, dtype=torch.bfloat16, kernel: str = "auto"):
    """(seg_len, nseg, m, sub) the library uses to split a prefill of this shape on one device."""
    plan = (ctypes.c_int64 * 4)()
    lib = _lib.load()
    _lib.check(lib.linattn_seq_plan(B, H, N, dk, dv, _DTYPES[dtype], _KERNELS[kernel], plan))
    return tuple(int(x) for x in plan)


@_on_tensor_device
def state_pass_segmented(k, v, log2g, seg_len: int, *, m: int = 1, nseg: int | None = None,
                         kernel: str = "auto", out=None):
    """Local end states of segments [p*seg_len, (p+1)*seg_len), each cut into m sub-segments.

    Returns [nseg*m, B, H, dk, dv] fp32 (each sub-segment from a zero state).
    """
    _require_cuda(k, v, log2g, out)
    _check_kv(k, v)
    B, H, N, dk = k.shape
    dv = v.shape[3]
    _check_log2g(log2g, H)
    if nseg is None:
        nseg = -(-N // seg_len)
    _check_state(out, (nseg * m, B, H, dk, dv), "out")
    if out is None:
        out = torch.empty((nseg * m, B, H, dk, dv), dtype=torch.float32, device=k.device)
    lib = _lib.load()
    _lib.check(lib.linattn_state_pass_segmented(k.data_ptr(), v.data_ptr(), out.data_ptr(), log2g.data_ptr(),
                                                B, H, N, dk, dv, _dtype_code(k), _KERNELS[kernel], seg_len,
                                                m, nseg, _stream()))
    return out


@_on_tensor_device
def segment_prefix(loc, loc_geom, seg_len: int, nseg: int, log2g, n: int, *, out=None):
    """Inclusive prefix states incl[p] at token min(n, (p+1)*seg_len), p < nseg, from the local
    states ``loc`` of ``state_pass_segmented`` (geometry ``loc_geom``); [nseg, B, H, dk, dv]."""
    _require_cuda(loc, log2g, out)
    _, B, H, dk, dv = loc.shape
    if out is None:
        out = torch.empty((nseg, B, H, dk, dv), dtype=torch.float32, device=loc.device)
    lib = _lib.load()
    _lib.check(lib.linattn_segment_prefix(loc.data_ptr(), loc_geom[0], loc_geom[1], loc.shape[0], out.data_ptr(),
                                          seg_len, nseg, log2g.data_ptr(), B, H, n, dk, dv, _stream()))
    return out


@_on_tensor_device
def prefill_segmented(q, k, v, log2g, seg_len: int, *, loc=None, loc_geom=None, inclusive: bool = False,
                      s_in=None, s_out=None, out=None, kernel: str = "auto"):
    """Prefill with every seg_len-token segment in parallel, seeded from s_in and ``loc``: local
    states from ``state_pass_segmented`` (geometry ``loc_geom = (seg_len, m)``), or, with
    ``inclusive``, prefix states from ``segment_prefix`` (one read per segment)."""
    _require_cuda(q, k, v, log2g, s_in, s_out, out, loc)
    _check_qkv(q, k, v)
    B, H, N, dk = q.shape
    dv = v.shape[3]
    _check_log2g(log2g, H)
    if out is None:
        out = torch.empty_like(v)
    if tuple(out.shape) != tuple(v.shape) or out.dtype != v.dtype:
        raise ShapeError(f"out must be {v.dtype} {tuple(v.shape)}, got {out.dtype} {tuple(out.shape)}")
    for st in (s_in, s_out):
        _check_state(st, (B, H, dk, dv))
    if loc is not None and (loc.dim() != 5 or tuple(loc.shape[1:]) != (B, H, dk, dv) or loc.dtype != torch.float32):
        raise ShapeError(f"loc must be float32 [n, B, H, dk, dv], got {loc.dtype} {tuple(loc.shape)}")
    lseg, lm = loc_geom if loc_geom is not None else (seg_len, 1)
    nloc = 0 if loc is None else loc.shape[0]
    lib = _lib.load()
    _lib.check(lib.linattn_prefill_segmented(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                             log2g.data_ptr(), _ptr(s_in), _ptr(s_out), _ptr(loc), lseg, lm,
                                             nloc, 1 if inclusive else 0, B, H, N, dk, dv, _dtype_code(q),
                                             _KERNELS[kernel], seg_len, _stream()))
    return out


@_on_tensor_device
def state_at(loc, loc_geom, pos: int, log2g, n: int, *, s_in=None, out=None):
    """gamma^pos s_in + sum over loc entries ending at or before pos of gamma^(pos - hi) loc[z]."""
    _require_cuda(loc, log2g, s_in, out)
    _, B, H, dk, dv = loc.shape
    if out is None:
        out = torch.empty((B, H, dk, dv), dtype=torch.float32, device=loc.device)
    lib = _lib.load()
    _lib.check(lib.linattn_state_at(loc.data_ptr(), loc_geom[0], loc_geom[1], loc.shape[0], _ptr(s_in),
                                    out.data_ptr(), pos, log2g.data_ptr(), B, H, n, dk, dv, _stream()))
    return out


@_on_tensor_device
def prefix_combine(gathered, seg_lens, rank: int, log2g, *, s_in=None):
    """Exclusive gamma-weighted prefix of gathered [P,B,H,dk,dv] end states."""
    _require_cuda(gathered, log2g, s_in)
    P, B, H, dk, dv = gathered.shape
    if s_in is None:
        s_in = torch.empty((B, H, dk, dv), dtype=torch.float32, device=gathered.device)
    lens = (ctypes.c_int64 * P)(*[int(x) for x in seg_lens])
    lib = _lib.load()
    _lib.check(lib.linattn_prefix_combine(gathered.data_ptr(), s_in.data_ptr(), lens, P, rank,
                                          log2g.data_ptr(), B, H, dk, dv, _stream()))
    return s_in


@_on_tensor_device
def decode_step(q, k, v, state, log2g, *, out=None):
    """S <- gamma S + k^T v ; o = q S for single tokens q,k [B,H,dk], v [B,H,dv]."""
    _require_cuda(q, k, v, state, log2g, out)
    if state.dtype != torch.float32:
        raise UsageError("decode state must be float32")
    _check_qkv(q, k, v, ndim=3)
    B, H, dk = q.shape
    dv = v.shape[-1]
    _check_log2g(log2g, H)
    if tuple(state.shape) != (B, H, dk, dv):
        raise ShapeError(f"state must be [B,H,dk,dv]={B, H, dk, dv}, got {tuple(state.shape)}")
    if out is None:
        out = torch.empty_like(v)
    if tuple(out.shape) != tuple(v.shape) or out.dtype != v.dtype:
        raise ShapeError(f"out must be {v.dtype} {tuple(v.shape)}, got {out.dtype} {tuple(out.shape)}")
    lib = _lib.load()
    _lib.check(lib.linattn_decode_step(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                       state.data_ptr(), log2g.data_ptr(), B, H, dk, dv,
                                       _dtype_code(q), _stream()))
    return out


@_on_tensor_device
def recurrent(q, k, v, log2g, *, s_in=None, s_out=None, out=None):
    """Row recurrence over whole sequences in one launch (S <- gamma S + k^T v; o = q S)."""
    _require_cuda(q, k, v, log2g, s_in, s_out, out)
    _check_qkv(q, k, v)
    B, H, N, dk = q.shape
    dv = v.shape[3]
    _check_log2g(log2g, H)
    for st in (s_in, s_out):
        _check_state(st, (B, H, dk, dv))
    if out is None:
        out = torch.empty_like(v)
    if tuple(out.shape) != tuple(v.shape) or out.dtype != v.dtype:
        raise ShapeError(f"out must be {v.dtype} {tuple(v.shape)}, got {out.dtype} {tuple(out.shape)}")
    lib = _lib.load()
    for b0, b1 in _batch_chunks(B, H):
        sl = (lambda t: None if t is None else t[b0:b1])   # noqa: E731
        _lib.check(lib.linattn_recurrent(q[b0:b1].data_ptr(), k[b0:b1].data_ptr(), v[b0:b1].data_ptr(),
                                         out[b0:b1].data_ptr(), log2g.data_ptr(), _ptr(sl(s_in)), _ptr(sl(s_out)),
                                         b1 - b0, H, N, dk, dv, _dtype_code(q), _stream()))
    return out


def prefill_kernel_name(dk: int, dv: int, dtype=torch.bfloat16, kernel: str = "auto") -> str:
    """Which kernel family a prefill of this shape runs: "prefill_tc" (tcgen05 bf16),
    "prefill_tf32" (tcgen05 3xTF32, the fp32 parity mode) or "prefill_simt" (FFMA)."""
    if kernel != "auto":
        return {"tc": "prefill_tc", "tf32": "prefill_tf32", "simt": "prefill_simt"}[kernel]
    code = _lib.load().linattn_prefill_kernel(dk, dv, _DTYPES[dtype])
    return {_lib.KERNEL_TC: "prefill_tc", _lib.KERNEL_TF32: "prefill_tf32"}.get(code, "prefill_simt")


def chunked_opcount(batch: int, heads: int, n: int, r: int, d: int, decay: bool, chunk: int) -> int:
    """Analytic two-level-block multiply-add count at chunk ``chunk`` (kernels.py:158-159, 164)."""
    total = 0
    full, rem = divmod(n, chunk)
    for length, count in ((chunk, full), (rem, 1 if rem else 0)):
        if decay:
            per = length * length * (r + d + 1) + 2 * length * r + 2 * length * r * d + r * d
        else:
            per = length * length * (r + d) + 2 * length * r * d
        total += per * count
    return total * batch * heads


def bytes_per_token_head(dk: int, dv: int, elem: int = 2) -> int:
    """Algorithmic prefill bytes per (token, head): q, k, v read once, o written once."""
    return elem * (2 * dk + 2 * dv)
