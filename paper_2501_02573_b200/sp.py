"""Sequence-parallel prefill across ranks (one process per GPU, NCCL over NVLink).

Algorithm (algebra = the reference recursion cross term,
kernels.py:185-189, with gamma^t * gamma^(mid-s) = gamma^(t+1) * gamma^(mid-1-s)):

  1. rank p owns the contiguous token segment [lo_p, hi_p) of length L_p;
     state pass (K4), split across the SMs: local states of sub-segments, combined into
     S_p = sum_t gamma^(L_p-1-t) k_t^T v_t from zero state;
  2. one all-gather of the fp32 end states [B, H, dk, dv] (the only exchange);
  3. prefix combine (K5): S_in(p) = sum_{q<p} gamma^(sum_{q<m<p} L_m) S_q;
  4. seeded chunked prefill of the segment from S_in(p) and the sub-segment states, every
     sub-segment in parallel.

Every rank computes only its own segment; the gathered states are tiny
(2 MiB per rank at H=32, d=128), so one collective suffices on NVSwitch.
The device operators come from a *backend* object; the product backend is the
CUDA library (``CudaBackend``).  Tests on CPU inject an explicit backend over
the gloo process group to exercise the host logic and the collective.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import ops


def segment_bounds(n: int, parts: int):
    """Contiguous, near-equal split of n tokens into ``parts`` segments."""
    base, extra = divmod(n, parts)
    bounds = [0]
    for p in range(parts):
        bounds.append(bounds[-1] + base + (1 if p < extra else 0))
    return [(bounds[p], bounds[p + 1]) for p in range(parts)]


class CudaBackend:
    """Product backend: the sm_100a kernels of liblinattn_b200.so.

    The local scan of a rank's segment is itself split across the SMs when batch x head
    leaves them idle (the same two-phase algebra inside the device, ``ops.seq_plan``): one
    state-only launch over every sub-segment, one prefix scan giving the state at each segment
    end (the last one is the rank's end state), one seeded launch over all segments.
    """

    def __init__(self, kernel: str = "auto"):
        self.kernel = kernel

    def local_states(self, k, v, log2g):
        """(opaque local data, this rank's end state [B, H, dk, dv] from a zero state)."""
        B, H, L, dk = k.shape
        dv = v.shape[3]
        seg, nseg, m, _ = ops.seq_plan(B, H, L, dk, dv, k.dtype, self.kernel)
        if nseg == 1:
            seg, m = L, 1
        else:
            # the state pass covers all nseg segments here: one wave of long CTAs beats more,
            # shorter ones once the units already fill most SMs
            sms = torch.cuda.get_device_properties(k.device).multi_processor_count
            if B * H * -(-dv // 128) * nseg >= 0.8 * sms:
                m = 1
        loc = ops.state_pass_segmented(k, v, log2g, seg, m=m, nseg=nseg, kernel=self.kernel)
        incl = ops.segment_prefix(loc, (seg, m), seg, nseg, log2g, L)
        return (incl, seg), incl[-1]

    def prefix_combine(self, gathered, seg_lens, rank, log2g):
        return ops.prefix_combine(gathered, seg_lens, rank, log2g)

    def prefill(self, q, k, v, log2g, s_in, local):
        incl, seg = local
        return ops.prefill_segmented(q, k, v, log2g, seg, loc=incl[:-1] if incl.shape[0] > 1 else None,
                                     loc_geom=(seg, 1), inclusive=True, s_in=s_in, kernel=self.kernel)


def sp_prefill(q_seg, k_seg, v_seg, log2g, seg_lens, group=None, backend=None):
    """Sequence-parallel prefill of this rank's segment.

    q_seg, k_seg: [B, H, L_p, dk]; v_seg: [B, H, L_p, dv] (this rank's tokens);
    seg_lens: list of every rank's segment length (same on all ranks).
    Returns this rank's output segment [B, H, L_p, dv].

    Per rank: one state pass over K, V (0.5x of the prefill bytes), one all-gather of a
    [B, H, dk, dv] fp32 state, one seeded prefill (1x) -- 1.5x the single-pass traffic.
    """
    backend = backend or CudaBackend()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if len(seg_lens) != world:
        raise ValueError(f"seg_lens has {len(seg_lens)} entries for world size {world}")
    if k_seg.shape[2] != seg_lens[rank]:
        raise ValueError(f"rank {rank} holds {k_seg.shape[2]} tokens, seg_lens says {seg_lens[rank]}")
    local_data, local = backend.local_states(k_seg, v_seg, log2g)   # end state from zero [B,H,dk,dv]
    if dist.is_initialized():   # the collective runs under any group (world 1 included: one code path)
        local = local.contiguous()
        # gloo has no device all-gather: stage through the host (CPU tests, shared-GPU path checks)
        host = local.is_cuda and dist.get_backend(group) == "gloo"
        src = local.cpu() if host else local
        flat = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                           device=src.device)
        dist.all_gather_into_tensor(flat, src, group=group)     # one collective; NCCL over NVLink
        gathered = flat.view((world,) + tuple(local.shape)).to(local.device)
    else:
        gathered = local[None]
    s_in = backend.prefix_combine(gathered, seg_lens, rank, log2g) if rank > 0 else None
    return backend.prefill(q_seg, k_seg, v_seg, log2g, s_in, local_data)
