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


# ---------------------------------------------------------------------------
# xi-slab decomposition of the macro loop (paper_2405_08764_b200/sharded.py):
# the sharded run equals the single-engine run bit for bit (restated oracle as
# the per-rank compute, gloo point-to-point for the halo columns).
# ---------------------------------------------------------------------------
def _shard_worker(rank, world, port, name, over, nsteps, out, deferred=False):
    import numpy as np
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Restated
    from paper_2405_08764_b200 import configs, sharded
    from paper_2405_08764_b200.engine import Problem

    O = Restated(threads=1)
    P = Problem(configs.copy_desc(configs.load(name)[0], **over))
    ed = P.engine_desc()
    sl = sharded.slabs(ed.Nxi, bool(ed.periodic_xi), world)[rank]
    sub = sharded.subset_desc(ed, sl)

    def step(U_in, U_out, t, bnd):
        st, o = O.projective_step(sub, U_in.numpy(), t, bnd)
        assert st == 0
        U_out.copy_(torch.from_numpy(o))

    runner = sharded.ShardedRun(sl, ed.Neta, step, dist, k=P.desc.k)
    U0 = torch.from_numpy(P.initial_field().reshape(-1).copy())
    dt = P.desc.T / P.desc.Nt
    if deferred:  # bench.py's loop: no per-step host round trip, one guard reduction at the end
        res = runner.run_deferred(U0, nsteps, dt, 0.0, P.boundary_table(0.0, nsteps))
        U, done, failed = res.U, res.steps_done, res.failed_step
    else:
        U, done, failed = runner.run(U0, nsteps, dt, 0.0, P.boundary_table(0.0, nsteps))
    full = runner.gather(U)
    out[rank] = (full.numpy().copy(), done, failed)
    dist.destroy_process_group()


@pytest.mark.parametrize("deferred", [False, True], ids=["per-step-guard", "deferred-guard"])
@pytest.mark.parametrize("name,over,world", [("c1_diffusion", {}, 2), ("c1_diffusion", {}, 3),
                                             ("c3_annulus", {}, 2), ("c3_annulus", {}, 3),
                                             ("c1_diffusion", {"dt_over_tau": 1000, "Nt": 50}, 2),
                                             ("c1_diffusion", {"dt_over_tau": 150, "Nt": 50}, 3)])
def test_sharded_run_equals_single_engine(name, over, world, deferred):
    import numpy as np

    from oracle.pyoracle import Restated
    from paper_2405_08764_b200 import configs
    from paper_2405_08764_b200.engine import Problem

    nsteps = 20 if "Nt" not in over else 50
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_shard_worker, args=(world, port, name, over, nsteps, out, deferred), nprocs=world, join=True)
        res = dict(out)
    P = Problem(configs.copy_desc(configs.load(name)[0], **over))
    ed = P.engine_desc()
    st, Uref, stats = Restated(threads=1).run(ed, P.initial_field(), nsteps, 0.0, P.boundary_table(0.0, nsteps))
    for r in range(world):
        U, done, failed = res[r]
        if st == 0:
            assert failed == 0 and done == nsteps
            assert np.array_equal(U.reshape(P.shape), Uref)
        else:  # the guard trips at the same macro step on every rank, with the same field
            assert failed == stats.failed_step and done == stats.steps_done
            if deferred:
                assert np.array_equal(U.reshape(P.shape), Uref)


@pytest.mark.parametrize("Nxi,periodic,world", [(19, False, 2), (19, False, 3), (128, True, 2), (128, True, 3),
                                                (8, True, 8), (8, False, 7), (64, True, 1)])
def test_peer_halo_links_cover_every_halo_once(Nxi, periodic, world):
    """The fused peer-memory halo (sharded.halo_links): every halo column a rank's
    3x3 stencils read (gaptooth.cpp:74-104, xi-wrap when periodic) is stored by
    exactly one link from its owner, into the counter side the rank waits on."""
    from paper_2405_08764_b200 import sharded

    sls = sharded.slabs(Nxi, periodic, world)
    owner = {i: s.rank for s in sls for i in range(s.i0, s.i1)}
    got = {r: [] for r in range(world)}
    for s in sls:
        for col, nb, side in sharded.halo_links(s):
            assert owner[col] == s.rank  # a rank only stores columns it computes
            got[nb].append((col, side))
    for s in sls:
        want = []
        if s.left() is not None:
            want.append((((s.i0 - 1) % Nxi) if periodic else s.i0 - 1, sharded.FROM_LEFT))
        if s.right() is not None:
            want.append(((s.i1 % Nxi) if periodic else s.i1, sharded.FROM_RIGHT))
        assert sorted(got[s.rank]) == sorted(want)
        assert sorted(sharded.incoming_sides(s)) == sorted(side for _, side in want)
        # halos that no link feeds are the global boundary columns (refresh_boundary)
        for h in ((s.i0 - 1), s.i1):
            if not periodic and h in (0, Nxi):
                assert all(c != h for c, _ in got[s.rank])
