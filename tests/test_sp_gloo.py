"""Sequence-parallel host logic over a real 2-rank process group (gloo, CPU).

The device operators are replaced by an explicit test backend built on the
CPU oracle; what is under test is sp.sp_prefill: segment bookkeeping, the one
all-gather of end states, and the rank-ordered prefix handoff.
"""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import linattn_oracle as orc


class OracleBackend:
    def __init__(self, gammas, decay=True):
        self.gammas = gammas
        self.decay = decay

    def local_states(self, k, v, log2g):
        s = np.stack([[orc.segment_end_state(k[x, h].numpy(), v[x, h].numpy(), self.gammas[h], self.decay)
                       for h in range(k.shape[1])] for x in range(k.shape[0])])
        return None, torch.from_numpy(s)

    def prefix_combine(self, gathered, seg_lens, rank, log2g):
        g = gathered.numpy()
        out = np.empty(g.shape[1:])
        for h in range(g.shape[2]):
            out[:, h] = orc.exclusive_prefix_states([g[p][:, h] for p in range(g.shape[0])], seg_lens,
                                                    self.gammas[h], self.decay)[rank]
        return torch.from_numpy(out)

    def prefill(self, q, k, v, log2g, s_in, local):
        out, _ = orc.seeded_blocked_attn(q.numpy(), k.numpy(), v.numpy(), self.gammas, self.decay,
                                         None if s_in is None else s_in.numpy(), block=16)
        return torch.from_numpy(out)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_02573_b200.sp import segment_bounds, sp_prefill
    b, c, v = orc.gen_inputs(2, 3, n, 5, 4, np.float64, 21)
    gammas = [0.0, 0.93, 1.0]
    bounds = segment_bounds(n, world)
    lens = [hi - lo for lo, hi in bounds]
    lo, hi = bounds[rank]
    seg = [torch.from_numpy(np.ascontiguousarray(x[:, :, lo:hi])) for x in (b, c, v)]
    out = sp_prefill(*seg, torch.zeros(3), lens, backend=OracleBackend(gammas))
    outs = [torch.empty(0)] * world
    dist.all_gather_object(outs, out)
    if rank == 0:
        full = torch.cat(outs, dim=2).numpy()
        ref = orc.oracle_attn(b, c, v, gammas, True)
        np.save(result_path, np.array([orc.max_rel_error(full, ref)]))
    dist.destroy_process_group()


def test_sp_prefill_two_ranks_gloo(tmp_path):
    for n in (97, 64):
        res = str(tmp_path / f"err{n}.npy")
        mp.spawn(_worker, args=(2, _free_port(), n, res), nprocs=2, join=True)
        assert float(np.load(res)[0]) <= 1e-12
