"""Multi-process plumbing of bench.py on CPU (gloo, world_size 2).

The hot path is single-GPU per north_star; bench.py --gpus N runs N
independent replicas (one process per GPU, weak scaling) and reports the
whole-job value = all ranks' updates / the MAX device time over ranks.  This
test exercises exactly that reduction with the gloo backend.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms = torch.tensor([10.0 + 5.0 * rank], dtype=torch.float64)  # each rank's device time
    dist.barrier()
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    updates_rank = 1_000_000
    value = world * updates_rank / (ms.item() * 1e-3)
    out[rank] = value
    dist.destroy_process_group()


def test_replica_value_uses_max_over_ranks():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        vals = dict(out)
    expect = world * 1_000_000 / (15.0e-3)
    assert vals[0] == pytest.approx(expect) and vals[1] == pytest.approx(expect)
