"""CPU oracle for the decayed causal linear-attention hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline``
/ ``--impl reference`` legs of ``bench.py`` may use it, and only as the
checker or as the timed CPU baseline -- never as a fallback for the GPU path.

This is a numpy restatement of the reference package ``linattn`` 0.1.0
(``/root/reference/pkg/src/linattn``; citations are relative to that tree).
Parity is PINNED: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by importing the reference itself in the
build container (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``),
plus the reference's own known-answer fixtures EX-A..EX-E
(``tests/conftest.py:7-51`` of the reference).

Conventions:
  * M[i, j] = gamma**(i - j) for i >= j else 0, with gamma**0 == 1 even when
    gamma == 0 (masks.py:22, masks.py:44-49).
  * decay=False means the binary causal mask; gamma is ignored.
  * Powers are built by repeated multiplication (masks.py:45-49), never pow().
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "decay_powers", "decay_mask", "oracle_attn", "blocked_attn", "row_recurrence",
    "segment_end_state", "exclusive_prefix_states", "sp_blocked_attn",
    "decode_steps", "max_rel_error", "gen_inputs", "log2_gamma", "bf16_round",
    "seeded_blocked_attn",
]


def decay_powers(gamma: float, first: int, count: int) -> np.ndarray:
    """f64 vector [gamma**first, gamma**(first+1), ...] of length ``count``.

    Restates ``decay_weights`` (masks.py:33-50): the running power starts at
    1.0, is multiplied ``first`` times, then once per emitted entry.
    """
    if count < 1:
        raise ValueError("count must be >= 1")
    w = 1.0
    for _ in range(first):
        w *= gamma
    out = np.empty(count, dtype=np.float64)
    for i in range(count):
        out[i] = w
        w *= gamma
    return out


def decay_mask(gamma: float, n: int, decay: bool = True) -> np.ndarray:
    """Dense f64 n x n lower-triangular mask (masks.py:53-64).

    Column j holds gamma**0, gamma**1, ... from the diagonal downwards, which
    is the same column-wise construction the reference uses.
    """
    m = np.zeros((n, n), dtype=np.float64)
    if not decay:
        return np.tril(np.ones((n, n), dtype=np.float64))
    col = decay_powers(gamma, 0, n)
    for j in range(n):
        m[j:, j] = col[: n - j]
    return m


def oracle_attn(b, c, v, gammas, decay: bool = True, out_dtype=None) -> np.ndarray:
    """Dense f64 (B C^T (.) M) V per (batch, head) slice (oracle.py:28-43).

    b, c: (batch, heads, N, r); v: (batch, heads, N, d); gammas: length heads.
    Returns f64 unless ``out_dtype`` is given (the reference casts back to the
    input dtype, oracle.py:42).
    """
    b = np.asarray(b)
    c = np.asarray(c)
    v = np.asarray(v)
    nb, nh, n, _ = b.shape
    out = np.empty(v.shape, dtype=np.float64)
    for h in range(nh):
        mask = decay_mask(float(gammas[h]), n, decay)
        for bi in range(nb):
            a = b[bi, h].astype(np.float64) @ c[bi, h].astype(np.float64).T
            out[bi, h] = (a * mask) @ v[bi, h].astype(np.float64)
    return out if out_dtype is None else out.astype(out_dtype)


def _blocked_slice(b, c, v, gamma, decay, block, dt, u0=None):
    """One (N, r) x (N, d) slice of the two-level block method.

    Restates ``_two_level_block_slice`` (kernels.py:139-166): per block of
    L <= ``block`` rows, intra = ((b c^T) (.) M_L) v, inter = (gamma^t b) u with
    t = 1..L, carry u <- gamma^L u + (gamma^(L-t) c)^T v.  Arithmetic runs in
    ``dt`` (the reference runs in the input dtype).  ``u0`` is an
    optional initial state (a new contract: the reference always starts at 0).
    Returns (out, final state).
    """
    n, r = b.shape
    d = v.shape[1]
    u = np.zeros((r, d), dtype=dt) if u0 is None else np.array(u0, dtype=dt)
    out = np.empty((n, d), dtype=dt)
    for s in range(0, n, block):
        e = min(s + block, n)
        L = e - s
        bi, ci, vi = b[s:e], c[s:e], v[s:e]
        if decay:
            m = decay_mask(gamma, L, True).astype(dt)
            w_in = decay_powers(gamma, 1, L).astype(dt)           # gamma^t, t=1..L
            w_out = decay_powers(gamma, 0, L)[::-1].astype(dt)    # gamma^(L-t)
            out[s:e] = ((bi @ ci.T) * m) @ vi + (w_in[:, None] * bi) @ u
            u = w_in[-1] * u + (w_out[:, None] * ci).T @ vi
        else:
            out[s:e] = ((bi @ ci.T) * np.tri(L, dtype=dt)) @ vi + bi @ u
            u = u + ci.T @ vi
    return out, u


def blocked_attn(b, c, v, gammas, decay: bool = True, block: int = 64,
                 dtype=None, slices=None):
    """Chunked linear-time attention over all (or a subset of) slices.

    This is the reference's "CPU blocking route" (kernels.py:139-166 driven by
    the batch x head loop of run_method, kernels.py:273-280).  ``slices``
    optionally restricts the work to a list of (batch, head) pairs (used for
    the bounded CPU-baseline sample); other outputs are left untouched (zero).
    """
    b = np.asarray(b)
    c = np.asarray(c)
    v = np.asarray(v)
    dt = np.dtype(dtype) if dtype is not None else v.dtype
    out = np.zeros(v.shape, dtype=dt)
    todo = slices if slices is not None else [
        (bi, h) for bi in range(b.shape[0]) for h in range(b.shape[1])]
    for bi, h in todo:
        o, _ = _blocked_slice(b[bi, h].astype(dt), c[bi, h].astype(dt),
                              v[bi, h].astype(dt), float(gammas[h]), decay, block, dt)
        out[bi, h] = o
    return out


def row_recurrence(b, c, v, gamma: float, decay: bool = True, u0=None, dtype=np.float64):
    """Per-token recurrence on one slice (kernels.py:93-106).

    u <- gamma u + c_i^T v_i ; o_i = b_i u  (decay applied before the update).
    Returns (out, final state).
    """
    n, r = b.shape
    d = v.shape[1]
    u = np.zeros((r, d), dtype=dtype) if u0 is None else np.array(u0, dtype=dtype)
    g = dtype(gamma) if decay else dtype(1.0)
    out = np.empty((n, d), dtype=dtype)
    for i in range(n):
        u = g * u + np.outer(c[i].astype(dtype), v[i].astype(dtype))
        out[i] = b[i].astype(dtype) @ u
    return out, u


def decode_steps(q, k, v, state, gammas, decay: bool = True):
    """Batched decode: apply the row recurrence token by token.

    q, k: (batch, heads, T, r); v: (batch, heads, T, d); state: (batch, heads,
    r, d) f64 initial state.  Returns (out f64, final state f64).
    """
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    s = np.array(state, dtype=np.float64)
    nb, nh, t, _ = q.shape
    out = np.empty(v.shape, dtype=np.float64)
    for h in range(nh):
        g = float(gammas[h]) if decay else 1.0
        for i in range(t):
            s[:, h] = g * s[:, h] + k[:, h, i, :, None] * v[:, h, i, None, :]
            out[:, h, i] = np.einsum("br,brd->bd", q[:, h, i], s[:, h])
    return out, s


def segment_end_state(c, v, gamma: float, decay: bool = True) -> np.ndarray:
    """End state of one segment scanned from zero, f64: sum_t gamma^(L-1-t) c_t^T v_t.

    This is the block carry (kernels.py:127-128) for a single block spanning
    the segment, equivalently the recursion's ``(w2 (.) C1)^T V1`` factor
    (kernels.py:187-188).
    """
    c = np.asarray(c, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    L = c.shape[0]
    w = decay_powers(gamma, 0, L)[::-1] if decay else np.ones(L)
    return (w[:, None] * c).T @ v


def exclusive_prefix_states(states, seg_lens, gamma: float, decay: bool = True):
    """S_in(p) = sum_{q<p} gamma^(sum_{q<m<p} L_m) S_q.

    Computed as the scan S_in(0) = 0, S_in(p) = gamma^L_{p-1} S_in(p-1) + S_{p-1}.
    """
    states = [np.asarray(s, dtype=np.float64) for s in states]
    acc = np.zeros_like(states[0])
    out = []
    for p, s in enumerate(states):
        out.append(acc.copy())
        carry = (gamma ** seg_lens[p]) if decay else 1.0
        acc = carry * acc + s
    return out


def sp_blocked_attn(b, c, v, gamma: float, parts: int, decay: bool = True, block: int = 64):
    """Sequence-parallel restatement on one slice, f64.

    Each part scans its contiguous segment from the prefix state it is given;
    the prefix comes from the zero-state segment end states through
    ``exclusive_prefix_states``.  Algebraically identical to the recursion's
    cross term (kernels.py:185-189): gamma^t * gamma^(mid-s) = gamma^(t+1) *
    gamma^(mid-1-s).
    """
    n = b.shape[0]
    bounds = np.linspace(0, n, parts + 1).astype(int)
    lens = [int(bounds[p + 1] - bounds[p]) for p in range(parts)]
    ends = [segment_end_state(c[bounds[p]:bounds[p + 1]], v[bounds[p]:bounds[p + 1]], gamma, decay)
            if lens[p] > 0 else np.zeros((b.shape[1], v.shape[1])) for p in range(parts)]
    prefix = exclusive_prefix_states(ends, lens, gamma, decay)
    out = np.empty((n, v.shape[1]), dtype=np.float64)
    for p in range(parts):
        lo, hi = bounds[p], bounds[p + 1]
        if hi > lo:
            out[lo:hi], _ = _blocked_slice(
                np.asarray(b[lo:hi], np.float64), np.asarray(c[lo:hi], np.float64),
                np.asarray(v[lo:hi], np.float64), gamma, decay, block, np.float64, u0=prefix[p])
    return out


def max_rel_error(out, ref) -> float:
    """max|out - ref| / max|ref| in f64 (verify.py:22-24)."""
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    denom = max(float(np.abs(ref).max()), np.finfo(np.float64).tiny)
    return float(np.abs(out - ref).max()) / denom


def gen_inputs(batch, heads, seqlen, rank, dim, dtype=np.float32, seed=0):
    """Seeded standard-normal (b, c, v) exactly as bench.py:77-84 draws them.

    PCG64 seeded with [seed, batch, heads, seqlen, rank, dim]; b, c, v drawn in
    that order.  Returns the three arrays (gamma is assigned by the caller).
    """
    rng = np.random.default_rng([seed, batch, heads, seqlen, rank, dim])
    b = rng.standard_normal((batch, heads, seqlen, rank)).astype(dtype)
    c = rng.standard_normal((batch, heads, seqlen, rank)).astype(dtype)
    v = rng.standard_normal((batch, heads, seqlen, dim)).astype(dtype)
    return b, c, v


def log2_gamma(gammas, decay: bool = True) -> np.ndarray:
    """f64-derived fp32 log2(gamma) per head; -inf for gamma == 0; 0 if no decay."""
    g = np.asarray(gammas, dtype=np.float64)
    if not decay:
        return np.zeros(g.shape, dtype=np.float32)
    with np.errstate(divide="ignore"):
        return np.log2(g).astype(np.float32)


def bf16_round(a) -> np.ndarray:
    """Round to the nearest bf16 (ties to even), returned as f32 (test helper)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def seeded_blocked_attn(b, c, v, gammas, decay: bool = True, s_in=None, block: int = 64):
    """Two-level block method over all slices in f64, optionally seeded with s_in [B,H,r,d].

    Returns (out [B,H,N,d], end state [B,H,r,d]) -- the contract of linattn_prefill.
    """
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    nb, nh = b.shape[:2]
    out = np.empty(v.shape, dtype=np.float64)
    end = np.empty((nb, nh, b.shape[3], v.shape[3]), dtype=np.float64)
    for x in range(nb):
        for h in range(nh):
            u0 = None if s_in is None else s_in[x, h]
            out[x, h], end[x, h] = _blocked_slice(b[x, h], c[x, h], v[x, h], float(gammas[h]), decay,
                                                  block, np.float64, u0=u0)
    return out, end
