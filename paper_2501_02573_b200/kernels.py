"""Method registry and ``run_method``: the drop-in boundary at run_method level.

The reference routes every method through ``run_method(method, inputs,
params, validate) -> (out, opcount)`` (kernels.py:257-281), looping over
(batch, head) slices.  This module keeps that signature and return contract
but each method here is ONE device launch over the whole (B, H, N, .) tensor:

=====================  =====================================================
``b200-chunked``       tcgen05 tensor-core chunked prefill, bf16 operands,
                       fp32 accumulation (replaces block-based /
                       two-level-block, kernels.py:109-166); tolerance 2e-2
``b200-chunked-f32``   the same algebra on the fp32 FFMA pipe (parity mode,
                       tolerance 1e-4 against the f64 oracle)
``b200-recurrent``     per-token recurrence through the decode-step kernel
                       (row-based semantics, kernels.py:93-106)
``b200-seqpar``        two-phase sequence-split prefill (state pass, prefix
                       combine, seeded prefill) over ``params.seq_parts``
                       segments on one device (recursion cross term,
                       kernels.py:185-189); the multi-GPU form is ``sp.py``
=====================  =====================================================

Output dtype equals input dtype; host (numpy) inputs are staged through the
device and returned as numpy, device (torch CUDA) inputs stay on the device.
There is no CPU fallback: without the CUDA library every method raises.
"""

from __future__ import annotations

import enum
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import LinAttnError, ResourceError, UsageError
from .tensor import (DEFER, AttnInputs, check_finite_all, check_output_then_inputs, finite_check_pending,
                     mark_finite, validate_inputs)

DEFAULT_MEM_CAP = 2 << 30  # kept for signature parity with the reference (oracle.py:16)
TC_CHUNK = 64      # token chunk of the bf16 tensor-core kernel (the reference default, kernels.py:57)
TF32_CHUNK = 32    # token chunk of the 3xTF32 tensor-core kernel (fp32 parity mode)
SIMT_CHUNK = 32    # token chunk of the FFMA kernel

REFERENCE_ONLY = ("vanilla", "row-based", "block-based", "recursion", "two-level-block",
                  "fleet", "fleet-tiled")


class MethodId(enum.Enum):
    B200_CHUNKED = "b200-chunked"
    B200_CHUNKED_F32 = "b200-chunked-f32"
    B200_RECURRENT = "b200-recurrent"
    B200_SEQPAR = "b200-seqpar"
    AUTO = "auto"

    @classmethod
    def parse(cls, name: str) -> "MethodId":
        """String -> MethodId, with the reference's UsageError on unknown names (kernels.py:35-41)."""
        for m in cls:
            if m.value == name:
                return m
        known = ", ".join(m.value for m in cls)
        if name in REFERENCE_ONLY:
            raise UsageError(f"method {name!r} is a CPU route of the reference package; "
                             f"this package provides the device methods ({known})")
        raise UsageError(f"unknown method {name!r} (known: {known})")


CONCRETE_METHODS = [m for m in MethodId if m is not MethodId.AUTO]


@dataclass
class BlockParams:
    """Tuning knobs (reference kernels.py:47-61 plus ``seq_parts``).

    ``block_size`` is the reference's block (chunk) length.  Each device kernel walks the
    sequence in chunks of a fixed length C (64 for the bf16 tensor-core kernel, 32 for the
    3xTF32 and FFMA kernels): a block of ``block_size = k * C`` tokens is exactly k consecutive
    kernel chunks -- the two-level block algebra is block-size invariant (reference
    test_kernels.py:114-124) -- so any positive multiple of C is honoured, and ``run_method``
    reports the opcount at C, the chunk actually used.  Other values raise UsageError.
    ``row_block``/``col_block``/``term_size``/``mem_cap`` feed reference-only routes and are
    accepted for signature parity.  ``seq_parts`` is the number of sequence segments for
    ``b200-seqpar``.
    """

    block_size: int = 64
    row_block: int = 64
    col_block: int | None = None
    term_size: int = 32
    mem_cap: int = DEFAULT_MEM_CAP
    seq_parts: int = 2


_COMPUTE = {
    MethodId.B200_CHUNKED: torch.bfloat16,
    MethodId.B200_CHUNKED_F32: torch.float32,
    MethodId.B200_RECURRENT: torch.float32,
    MethodId.B200_SEQPAR: torch.bfloat16,
}


_INT64_MAX = (1 << 63) - 1
_NF_SLOTS = threading.local()


def _nonfinite_slot(device) -> torch.Tensor:
    """A per-thread, per-device int64 verdict slot reset to INT64_MAX on the current stream."""
    slots = getattr(_NF_SLOTS, "d", None)
    if slots is None:
        slots = _NF_SLOTS.d = {}
    slot = slots.get(device)
    if slot is None:   # a clean verdict leaves the slot at INT64_MAX: it is reset only after a hit
        slot = slots[device] = torch.full((1,), _INT64_MAX, dtype=torch.int64, device=device)
    return slot


def kernel_chunk(method: MethodId, inputs: AttnInputs) -> int:
    """Token chunk of the kernel ``method`` runs for these inputs (1 for the row recurrence)."""
    if method is MethodId.B200_RECURRENT:
        return 1
    cdt = _COMPUTE[method]
    name = ops.prefill_kernel_name(inputs.rank, inputs.dim, cdt)
    return {"prefill_tc": TC_CHUNK, "prefill_tf32": TF32_CHUNK}.get(name, SIMT_CHUNK)


def _check_block_size(method: MethodId, params: "BlockParams", chunk: int) -> None:
    bs = params.block_size
    if method is MethodId.B200_RECURRENT or bs is None:
        return
    if not isinstance(bs, (int, np.integer)) or bs < 1 or bs % chunk:
        raise UsageError(f"{method.value} runs chunks of {chunk} tokens for these inputs: block_size must "
                         f"be a positive multiple of {chunk} (got {bs!r})")


def _to_device(x, dtype):
    """Device (CUDA) tensors only: host inputs go through ``_host_pipelined``."""
    return x.to(dtype=dtype).contiguous()


def _seqpar(q, k, v, log2g, parts: int, kernel: str):
    """Two-phase sequence split on one device: segment-local state pass, then every segment
    seeded from the earlier ones and run in parallel (recursion cross term, kernels.py:185-189)."""
    return ops.prefill(q, k, v, log2g, kernel=kernel, seq_split=max(1, parts))


def _recurrent(q, k, v, log2g):
    """Row-based route (kernels.py:93-106): one launch walks every token with the state on chip.
    Rows that are not a multiple of 16 bytes are zero-padded to one (zero k columns leave the
    extra state rows at zero, the extra v columns are dropped); only dk > 256, past the scan
    kernel's state budget, steps the decode kernel per token."""
    B, H, N, dk = q.shape
    dv = v.shape[3]
    ev = 16 // q.element_size()
    if dk <= 256:
        if dk % ev == 0 and dv % ev == 0:
            return ops.recurrent(q, k, v, log2g)
        pk, pv = -(-dk // ev) * ev - dk, -(-dv // ev) * ev - dv
        pad = torch.nn.functional.pad
        out = ops.recurrent(pad(q, (0, pk)), pad(k, (0, pk)), pad(v, (0, pv)), log2g)
        return out[..., :dv].contiguous()
    state = torch.zeros((B, H, dk, dv), dtype=torch.float32, device=q.device)
    out = torch.empty_like(v)
    for i in range(N):
        out[:, :, i] = ops.decode_step(q[:, :, i].contiguous(), k[:, :, i].contiguous(),
                                       v[:, :, i].contiguous(), state, log2g)
    return out


def _pieces(batch: int, heads: int, target: int = 16):
    """Independent (batch, head-range) pieces for host<->device overlap, about `target` of them.

    Each piece is one batch index and a contiguous head range (contiguous in [B, H, N, d]),
    so the first H2D and the last D2H -- the parts no overlap can hide -- shrink to 1/target.
    """
    per_b = max(1, min(heads, -(-target // batch)))          # head groups per batch index
    edges = [round(i * heads / per_b) for i in range(per_b + 1)]
    return [(slice(b, b + 1), slice(edges[i], edges[i + 1])) for b in range(batch) for i in range(per_b)]


# (dtype, slot, role) -> pinned host buffer, grown on demand and kept across calls (page-locking
# is slow); per thread, so concurrent run_method calls never share a staging buffer (the
# reference's calls are reentrant)
_STAGING = threading.local()


_COPY_POOL = None


def _host_copy(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst.copy_(src) on the host, spread over the available cores when torch itself runs
    single-threaded (torchrun sets OMP_NUM_THREADS=1); torch releases the GIL while copying."""
    global _COPY_POOL
    workers = min(len(os.sched_getaffinity(0)), 16)
    if torch.get_num_threads() > 1 or workers <= 1 or dst.numel() < (1 << 21):
        dst.copy_(src)
        return
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _COPY_POOL = ThreadPoolExecutor(max_workers=workers, thread_name_prefix="linattn-copy")
    d, s_ = dst.view(-1), src.reshape(-1)
    step = -(-d.numel() // workers)
    futures = [_COPY_POOL.submit(d[a:a + step].copy_, s_[a:a + step]) for a in range(0, d.numel(), step)]
    for f in futures:
        f.result()


def release_staging_buffers() -> None:
    """Free the calling thread's cached pinned staging buffers (host-input ``run_method`` calls
    keep up to eight piece-sized page-locked buffers per thread for reuse) and return the
    library's cached device workspace (sequence-split / balanced-schedule pools) to the driver."""
    _STAGING.__dict__.pop("bufs", None)
    if torch.cuda.is_available():
        from . import _lib
        lib = _lib.load()
        torch.cuda.synchronize()           # pool frees are stream-ordered
        _lib.check(lib.linattn_release_workspace())


def _staging(dtype, slot: int, role: int, numel: int) -> torch.Tensor:
    """A pinned host buffer of at least ``numel`` elements, private to the calling thread."""
    cache = getattr(_STAGING, "bufs", None)
    if cache is None:
        cache = _STAGING.bufs = {}
    key = (dtype, slot, role)
    buf = cache.get(key)
    if buf is None or buf.numel() < numel:
        buf = torch.empty(numel, dtype=dtype).pin_memory()
        cache[key] = buf
    return buf[:numel]


def _host_pipelined(inputs: AttnInputs, cdt, run, result, pieces: int = 16):
    """Host tensors through the device in pieces: H2D(i+1) | prefill(i) | D2H(i-1) overlap.

    Every (batch, head) slice is independent (kernels.py:273-280), so the batch is cut into
    pieces on the batch axis (or the head axis when B == 1) and each piece runs on three
    streams -- copy-in, compute (torch's current stream), copy-out -- ordered by events.
    With pinned host buffers both PCIe directions and the kernel run concurrently.

    Pageable sources (numpy arrays, the reference's own calling convention) go through a
    two-slot ring of pinned staging buffers in the COMPUTE dtype: the host copy into slot i%2
    (multi-threaded, converting f64/f32 -> compute dtype on the way, so fewer bytes cross PCIe)
    overlaps the DMA of the other slot; results come back in the compute dtype and are widened
    while they are copied out of their pinned slot.
    """
    numpy_in = not isinstance(inputs.v, torch.Tensor)
    b, c, v = (torch.from_numpy(np.ascontiguousarray(x)) if not isinstance(x, torch.Tensor) else x
               for x in (inputs.b, inputs.c, inputs.v))
    in_dtype = v.dtype
    dev = torch.device("cuda", torch.cuda.current_device())
    qd = torch.empty(b.shape, dtype=cdt, device=dev)
    kd = torch.empty(c.shape, dtype=cdt, device=dev)
    vd = torch.empty(v.shape, dtype=cdt, device=dev)
    od = torch.empty(v.shape, dtype=cdt, device=dev)
    if result is None:
        result = torch.empty(v.shape, dtype=in_dtype)
    elif not isinstance(result, torch.Tensor):
        result = torch.from_numpy(result)
    staged_in = not all(x.is_pinned() for x in (b, c, v))
    staged_out = not result.is_pinned()
    log2g = ops.log2_gamma(inputs.gamma, inputs.decay, device=dev)
    compute = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    s_in.wait_stream(compute)          # device buffers were allocated on the compute stream
    slot_loaded = [None, None]         # H2D of the piece last staged in each slot
    pending = None                     # (event, pinned slice, result view) still to copy out
    for i, (bs, hs) in enumerate(_pieces(v.shape[0], v.shape[1], pieces)):
        slot = i % 2
        loaded = torch.cuda.Event()
        if staged_in and slot_loaded[slot] is not None:
            slot_loaded[slot].synchronize()                # its previous DMA has read the slot
        with torch.cuda.stream(s_in):
            for role, (host, d) in enumerate(((b, qd), (c, kd), (v, vd))):
                src = host[bs, hs]
                if staged_in:
                    stg = _staging(cdt, slot, role, src.numel()).view(src.shape)
                    _host_copy(stg, src)                     # host copy + cast, all cores
                    d[bs, hs].copy_(stg, non_blocking=True)
                elif src.dtype == cdt:
                    d[bs, hs].copy_(src, non_blocking=True)
                else:   # pinned, other dtype: stage in the host dtype, cast on the device
                    d[bs, hs].copy_(src.to(device=dev, non_blocking=True))
            loaded.record(s_in)
        slot_loaded[slot] = loaded
        compute.wait_event(loaded)
        run(qd[bs, hs], kd[bs, hs], vd[bs, hs], log2g[hs], od[bs, hs])
        computed = torch.cuda.Event()
        computed.record(compute)
        done = torch.cuda.Event()
        with torch.cuda.stream(s_out):
            s_out.wait_event(computed)
            if staged_out:
                ostg = _staging(cdt, slot, 3, od[bs, hs].numel()).view(od[bs, hs].shape)
                ostg.copy_(od[bs, hs], non_blocking=True)
            else:
                src = od[bs, hs] if in_dtype == cdt else od[bs, hs].to(in_dtype)
                result[bs, hs].copy_(src, non_blocking=True)
            done.record(s_out)
        if pending is not None:                            # previous piece: widen into result
            pending[0].synchronize()
            _host_copy(pending[2], pending[1])
            pending = None
        if staged_out:
            pending = (done, ostg, result[bs, hs])
    if pending is not None:
        pending[0].synchronize()
        _host_copy(pending[2], pending[1])
    s_out.synchronize()
    return result.numpy() if numpy_in else result


def run_method(method: MethodId, inputs: AttnInputs, params: BlockParams | None = None,
               validate: bool = True, out=None):
    """Run a concrete device method; returns (output, analytic opcount) (kernels.py:257-281).

    ``out`` (optional, not in the reference signature) is a caller-owned result
    buffer of the input's shape and dtype -- e.g. a pinned host tensor, so the
    device->host copy of a host-tensor call runs at full PCIe bandwidth.
    Device memory exhaustion raises the reference's ``ResourceError`` (errors.py:25; the
    reference raises it when a buffer would exceed its byte cap), so ``run_bench`` records an
    OOM row and carries on exactly as it does for the reference's capped methods.
    """
    try:
        return _run_method(method, inputs, params, validate, out)
    except torch.OutOfMemoryError as exc:
        raise ResourceError(f"device memory exhausted running {method}: {str(exc).splitlines()[0]}") from exc


def _run_method(method, inputs, params, validate, out):
    if isinstance(method, str):
        method = MethodId.parse(method)
    if method is MethodId.AUTO:
        raise UsageError("auto must be resolved by dispatch.decode, not run_method")
    if params is None:
        params = BlockParams()
    if validate:
        validate_inputs(inputs, check_values=DEFER)   # CUDA inputs: checked through the output below
    cdt = _COMPUTE[method]
    chunk = kernel_chunk(method, inputs)
    _check_block_size(method, params, chunk)
    host = not inputs.on_device
    torch_host = inputs.on_device and not inputs.v.is_cuda
    in_dtype = inputs.v.dtype
    if torch_host or host:
        # host tensors: (batch, head) pieces through the overlapped copy/compute pipeline
        if not torch.cuda.is_available():
            raise LinAttnError("no CUDA device: the B200 path has no CPU fallback")
        if method is MethodId.B200_RECURRENT:
            def run(q, k, v, l2, o):
                ev = 16 // q.element_size()
                if q.shape[3] % ev == 0 and v.shape[3] % ev == 0 and q.shape[3] <= 256:
                    ops.recurrent(q, k, v, l2, out=o)
                else:
                    o.copy_(_recurrent(q, k, v, l2))
            ops_count = inputs.batch * inputs.heads * inputs.seqlen * inputs.rank * inputs.dim * (
                3 if inputs.decay else 2)  # reference row-based count (kernels.py:105)
        else:
            kernel = "auto"
            split = max(1, int(params.seq_parts)) if method is MethodId.B200_SEQPAR else None
            run = lambda q, k, v, l2, o: ops.prefill(q, k, v, l2, out=o, kernel=kernel, seq_split=split)  # noqa: E731
            ops_count = ops.chunked_opcount(inputs.batch, inputs.heads, inputs.seqlen, inputs.rank,
                                            inputs.dim, inputs.decay, chunk)
        # the row recurrence is one serial chain per (b, h): few, wide pieces keep the SMs busy
        pieces = 2 if method is MethodId.B200_RECURRENT else 16
        return _host_pipelined(inputs, cdt, run, out, pieces), ops_count
    q = _to_device(inputs.b, cdt)
    k = _to_device(inputs.c, cdt)
    v = _to_device(inputs.v, cdt)
    log2g = ops.log2_gamma_cached(inputs.gamma, inputs.decay, q.device)
    fused_check = validate and finite_check_pending(inputs) and method is not MethodId.B200_RECURRENT
    if method in (MethodId.B200_CHUNKED, MethodId.B200_CHUNKED_F32) and fused_check:
        # the entry contract's NaN/Inf check rides on the launch (fused into the bf16 tensor-core
        # epilogue); the inputs are rescanned only if the output is not clean
        slot = _nonfinite_slot(q.device)
        out_dev = ops.prefill(q, k, v, log2g, kernel="auto", nonfinite=slot)
        if int(slot.item()) != _INT64_MAX:
            slot.fill_(_INT64_MAX)
            check_finite_all((("B", inputs.b), ("C", inputs.c), ("V", inputs.v)))
        mark_finite(inputs)
    elif method in (MethodId.B200_CHUNKED, MethodId.B200_CHUNKED_F32):
        out_dev = ops.prefill(q, k, v, log2g, kernel="auto")
    elif method is MethodId.B200_SEQPAR:
        out_dev = _seqpar(q, k, v, log2g, max(1, int(params.seq_parts)), "auto")
    else:
        out_dev = _recurrent(q, k, v, log2g)
    if validate:
        check_output_then_inputs(inputs, out_dev)
    ops_count = ops.chunked_opcount(inputs.batch, inputs.heads, inputs.seqlen, inputs.rank,
                                    inputs.dim, inputs.decay, chunk)
    if method is MethodId.B200_RECURRENT:
        ops_count = inputs.batch * inputs.heads * inputs.seqlen * inputs.rank * inputs.dim * (
            3 if inputs.decay else 2)  # reference row-based count (kernels.py:105)
    if out is not None:
        out.copy_(out_dev)
        return out, ops_count
    return out_dev.to(in_dtype), ops_count
