"""Sequence parallelism with real processes and the device kernels (one GPU shared by 2 ranks).

Each rank runs sp.sp_prefill with the CUDA backend on its own token segment; the one
collective (all-gather of [B, H, dk, dv] fp32 end states) runs over a gloo group (NCCL needs
one GPU per rank, and the test box has one).  The concatenated outputs must match the f64
oracle -- the same algebra the NCCL path runs on 8 GPUs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import linattn_oracle as orc

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2501_02573_b200 import ops
    from paper_2501_02573_b200.sp import segment_bounds, sp_prefill
    b, c, v = orc.gen_inputs(1, 3, n, 128, 128, np.float32, 23)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    gam = [1 - 2.0 ** -6, 1 - 2.0 ** -13, 0.0]
    bounds = segment_bounds(n, world)
    lens = [hi - lo for lo, hi in bounds]
    lo, hi = bounds[rank]
    seg = [torch.from_numpy(np.ascontiguousarray(x[:, :, lo:hi])).to("cuda", torch.bfloat16) for x in (b, c, v)]
    out = sp_prefill(*seg, ops.log2_gamma(gam, True, "cuda"), lens).float().cpu()
    outs = [None] * world
    dist.all_gather_object(outs, out)
    if rank == 0:
        full = torch.cat(outs, dim=2).numpy()
        np.save(result_path, np.array([orc.max_rel_error(full, orc.oracle_attn(b, c, v, gam, True))]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 6000), (3, 4097)])
def test_sp_prefill_processes_on_device(tmp_path, world, n):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res = str(tmp_path / "err.npy")
    mp.spawn(_worker, args=(world, _free_port(), n, res), nprocs=world, join=True)
    assert float(np.load(res)[0]) <= 2e-2


def _nccl_worker(rank, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    from paper_2501_02573_b200 import ops
    from paper_2501_02573_b200.sp import sp_prefill
    b, c, v = orc.gen_inputs(1, 4, 5000, 128, 128, np.float32, 29)
    b, c, v = orc.bf16_round(b), orc.bf16_round(c), orc.bf16_round(v)
    gam = [1 - 2.0 ** -6, 1 - 2.0 ** -13, 0.5, 1.0]
    x = [torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.bfloat16) for a in (b, c, v)]
    out = sp_prefill(*x, ops.log2_gamma(gam, True, "cuda"), [5000]).float().cpu().numpy()
    np.save(result_path, np.array([orc.max_rel_error(out, orc.oracle_attn(b, c, v, gam, True))]))
    dist.destroy_process_group()


def test_sp_prefill_nccl_group(tmp_path):
    """The NCCL code path of sp_prefill (all_gather_into_tensor of the fp32 end states on the
    device, no host staging) on a one-rank NCCL group: the box has one GPU and NCCL allows one
    rank per device, so this is the largest NCCL group a test can build here."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res = str(tmp_path / "err.npy")
    mp.spawn(_nccl_worker, args=(_free_port(), res), nprocs=1, join=True)
    assert float(np.load(res)[0]) <= 2e-2
