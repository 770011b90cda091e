"""Prefill -> decode state handoff and the per-token decode API.

The reference has no state input/output: every method starts from U = 0
(kernels.py:97, 114, 144).  Serving needs the prefill to hand its end state to
a per-token decoder, so this module adds that contract:

    out, state = prefill_with_state(inputs)      # state: RecurrentState
    o_t = state.step(q_t, k_t, v_t)             # S <- gamma S + k^T v ; o = q S

State layout: one fp32 [B, H, dk, dv] tensor in HBM, row-major (dv fastest),
so the decode kernel streams it with 128-bit coalesced accesses.  Continuity
is exact in the algebra: decoding token N+1.. after a prefill of N tokens
equals the oracle on the concatenated sequence (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import torch

from . import ops
from .errors import ShapeError, UsageError
from .tensor import AttnInputs, validate_inputs


class RecurrentState:
    """fp32 decode state [B, H, dk, dv] plus the per-head log2(gamma)."""

    def __init__(self, batch: int, heads: int, rank: int, dim: int, gamma, decay: bool = True,
                 device="cuda", state: torch.Tensor | None = None):
        gamma = [float(g) for g in (gamma if not isinstance(gamma, (int, float)) else [gamma] * heads)]
        if len(gamma) != heads:
            raise ShapeError(f"gamma must have one entry per head ({heads}), got {len(gamma)}")
        self.gamma = gamma
        self.decay = decay
        self.log2g = ops.log2_gamma(gamma, decay, device=device)
        if state is None:
            state = torch.zeros((batch, heads, rank, dim), dtype=torch.float32, device=device)
        if tuple(state.shape) != (batch, heads, rank, dim) or state.dtype != torch.float32:
            raise ShapeError("state must be float32 [batch, heads, rank, dim]")
        self.state = state.contiguous()

    @property
    def shape(self):
        return tuple(self.state.shape)

    def step(self, q, k, v, out=None):
        """One token per (b, h): q, k [B,H,dk] (or [B,H,1,dk]); v [B,H,dv]."""
        squeeze = q.dim() == 4
        if squeeze:
            q, k, v = q[:, :, 0], k[:, :, 0], v[:, :, 0]
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        if not (q.dtype == k.dtype == v.dtype):
            raise UsageError("q, k, v must share a dtype")
        o = ops.decode_step(q, k, v, self.state, self.log2g, out=out)
        return o[:, :, None] if squeeze else o

    def clone(self) -> "RecurrentState":
        return RecurrentState(self.shape[0], self.shape[1], self.shape[2], self.shape[3],
                              self.gamma, self.decay, self.state.device, self.state.clone())


def prefill_with_state(inputs: AttnInputs, kernel: str = "auto", s_in: RecurrentState | None = None):
    """Chunked prefill on device inputs returning (out, RecurrentState at the end)."""
    validate_inputs(inputs)
    if not inputs.on_device:
        raise UsageError("prefill_with_state takes device tensors (see run_method for host arrays)")
    st = RecurrentState(inputs.batch, inputs.heads, inputs.rank, inputs.dim, inputs.gamma,
                        inputs.decay, inputs.b.device)
    out = ops.prefill(inputs.b, inputs.c, inputs.v, st.log2g,
                      s_in=None if s_in is None else s_in.state, s_out=st.state, kernel=kernel)
    return out, st
