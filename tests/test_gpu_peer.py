"""Decomposed run with the fused peer-memory halo (pd_projective_step_halo,
sharded.PeerRun): every rank's step kernel stores its edge
columns straight into the neighbours' field buffers and bumps their link
counters; the ranks' streams wait on their own counters (stream memory
operations, nothing spins).  The result must equal the single-engine run bit
for bit (every patch value is computed from the same stencil values with the
same arithmetic), including where the blow-up guard trips (cpi.cpp:187-202).

On one GPU the ranks are either engines on separate streams of one process
(pointers used directly) or separate processes mapping each other's buffers
through CUDA IPC — the transport bench.py --gpus N uses across GPUs.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2405_08764_b200 import abi, configs, sharded
from paper_2405_08764_b200.engine import Engine, Problem

pytestmark = pytest.mark.gpu

FAST, EXACT = abi.PD_MODE_FAST, abi.PD_MODE_EXACT


def assemble(results, slabs, shape, periodic):
    """Full field from each rank's own columns (the boundary is refreshed alike on every rank)."""
    full = results[0].reshape(shape).copy()
    for U, sl in zip(results, slabs):
        full[sl.i0:sl.i1] = U.reshape(shape)[sl.i0:sl.i1]
    if periodic:
        full[-1] = full[0]
    return full


CASES = [("c1_diffusion", {}, 2), ("c1_diffusion", {}, 3), ("c3_annulus", {}, 2), ("c3_annulus", {}, 3),
         ("c2_cdr_tanh", {}, 4), ("c4_shear", {"N_xi": 65, "N_eta": 33, "Nt": 10}, 3),
         ("c1_diffusion", {"dt_over_tau": 1000, "Nt": 50}, 2), ("c1_diffusion", {"dt_over_tau": 150, "Nt": 50}, 3)]


@pytest.mark.parametrize("name,over,world", CASES,
                         ids=[f"{n}-{'-'.join(f'{k}{v}' for k, v in o.items()) or 'base'}-w{w}" for n, o, w in CASES])
@pytest.mark.parametrize("mode", [EXACT, FAST], ids=["exact", "fast"])
def test_peer_halo_run_equals_single_engine(name, over, world, mode, gpu):
    import torch

    P = Problem(configs.copy_desc(configs.load(name)[0], **over))
    ed = P.engine_desc()
    nsteps = min(20, P.desc.Nt) if "Nt" not in over else P.desc.Nt
    periodic = bool(ed.periodic_xi)
    sls = sharded.slabs(ed.Nxi, periodic, world)
    dev = torch.device("cuda", 0)
    engines = [Engine(sharded.subset_desc(ed, sl), mode) for sl in sls]
    assert sum(E.P for E in engines) == P.engine_desc().npatches
    runners = sharded.local_peer_group(engines, sls, ed.Neta, dev)
    U0 = torch.from_numpy(P.initial_field().reshape(-1).copy()).to(dev)
    bnd = P.boundary_table(0.0, nsteps)
    res = sharded.run_peer(runners, [U0] * world, nsteps, P.desc.T / P.desc.Nt, 0.0, bnd)
    full = assemble([r.U.cpu().numpy() for r in res], sls, P.shape, periodic)

    E = Engine.from_problem(P, mode=mode)
    Uref, stats = E.run(P.initial_field(), nsteps, bnd=bnd, raise_on_instability=False)
    failed = stats.failed_step  # 0, or the macro step whose guard tripped (the field is the one after it)
    for r in res:
        assert r.failed_step == failed
        if not failed:
            assert r.steps_done == nsteps
    assert np.array_equal(full, Uref)


def test_peer_halo_second_run_reuses_counters(gpu):
    """Counters are cumulative over a runner's life: two consecutive runs on the
    same group (the bench's warm-up + timed runs) both equal the single engine."""
    import torch

    P = Problem(configs.load("c3_annulus")[0])
    ed = P.engine_desc()
    sls = sharded.slabs(ed.Nxi, True, 2)
    dev = torch.device("cuda", 0)
    runners = sharded.local_peer_group([Engine(sharded.subset_desc(ed, sl), FAST) for sl in sls], sls, ed.Neta, dev)
    U0 = torch.from_numpy(P.initial_field().reshape(-1).copy()).to(dev)
    dt = P.desc.T / P.desc.Nt
    E = Engine.from_problem(P, mode=FAST)
    for nsteps in (7, 12):
        res = sharded.run_peer(runners, [U0] * 2, nsteps, dt)
        Uref, _ = E.run(P.initial_field(), nsteps)
        assert np.array_equal(assemble([r.U.cpu().numpy() for r in res], sls, P.shape, True), Uref)
    assert all(r.steps_total == 19 for r in runners)


def test_peer_halo_argument_checks(gpu):
    import ctypes as C

    import torch

    from paper_2405_08764_b200.engine import lib

    P = Problem(configs.load("c1_diffusion")[0])
    E = Engine.from_problem(P, mode=FAST)
    dev = torch.device("cuda", 0)
    X = torch.zeros(2, P.shape[0] * P.shape[1], dtype=torch.float64, device=dev)
    h = abi.HaloOut()
    h.nlinks = 3
    L = lib()
    assert L.pd_projective_step_halo(E.h, X[0].data_ptr(), X[1].data_ptr(), 0.0, None, None, C.byref(h)) == \
        abi.PD_VALIDATION_ERROR
    h.nlinks = 1
    h.column[0] = 1
    assert L.pd_projective_step_halo(E.h, X[0].data_ptr(), X[1].data_ptr(), 0.0, None, None, C.byref(h)) == \
        abi.PD_VALIDATION_ERROR  # no destination / counter
    h.nlinks = 0
    assert L.pd_projective_step_halo(E.h, X[0].data_ptr(), X[0].data_ptr(), 0.0, None, None, C.byref(h)) == \
        abi.PD_VALIDATION_ERROR  # in place
    assert L.pd_stream_wait_flag(E.h, None, 1) == abi.PD_VALIDATION_ERROR


# ---------------------------------------------------------------------------
# one process per rank, buffers shared through CUDA IPC (bench.py --gpus N's
# transport); here both processes sit on GPU 0 and gloo carries the handles
# and the one guard reduction
# ---------------------------------------------------------------------------
def _ipc_worker(rank, world, port, name, over, mode, nsteps, out):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = Problem(configs.copy_desc(configs.load(name)[0], **over))
    ed = P.engine_desc()
    sl = sharded.slabs(ed.Nxi, bool(ed.periodic_xi), world)[rank]
    dev = torch.device("cuda", 0)
    E = Engine(sharded.subset_desc(ed, sl), mode)
    run = sharded.peer_runner(E, sl, ed.Neta, dist, dev, k=ed.k)

    def red(x):
        t = x.detach().cpu().clone()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t

    U0 = torch.from_numpy(P.initial_field().reshape(-1).copy()).to(dev)
    res = sharded.run_peer([run], [U0], nsteps, P.desc.T / P.desc.Nt, reduce_max=red, barrier=dist.barrier)[0]
    full = sharded.ShardedRun(sl, ed.Neta, None, dist, stage_cpu=True).gather(res.U.clone())
    out[rank] = (full.cpu().numpy(), res.steps_done, res.failed_step)
    dist.barrier()
    sharded.close_peer_runner(run)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,over,world", [("c3_annulus", {}, 2), ("c4_shear", {"N_xi": 65, "N_eta": 33, "Nt": 8}, 3),
                                             ("c1_diffusion", {"k": 1}, 2)],
                         ids=["c3-w2", "c4-small-w3", "c1-k1-w2"])
def test_peer_halo_ipc_processes_equal_single_engine(name, over, world, gpu):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    P = Problem(configs.copy_desc(configs.load(name)[0], **over))
    nsteps = min(12, P.desc.Nt)
    with mp.Manager() as m:
        out = m.dict()
        ctx = mp.spawn(_ipc_worker, args=(world, port, name, over, FAST, nsteps, out), nprocs=world, join=False)
        for _ in range(600):  # bounded: a lost counter would leave a stream waiting
            if ctx.join(timeout=1):
                break
        else:
            for p in ctx.processes:
                p.kill()
            pytest.fail("IPC peer-halo run did not finish in 600 s")
        res = dict(out)
    E = Engine.from_problem(P, mode=FAST)
    Uref, _ = E.run(P.initial_field(), nsteps)
    for r in range(world):
        U, done, failed = res[r]
        assert failed == 0 and done == nsteps
        assert np.array_equal(U.reshape(P.shape), Uref)


def test_bench_multi_rank_path_runs_peer_exchange(gpu):
    """bench.py --gpus 2 under torchrun, both ranks on GPU 0 (PD_BENCH_ONE_DEVICE,
    gloo for the collectives): the N > 1 code path runs end to end through the
    fused peer-memory halo and prints one line from rank 0."""
    import json
    import os
    import socket
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, PD_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(root / "bench.py"),
           "--gpus", "2", "--steps", "4", "--warmup", "3", "--config", "c3_annulus"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["steps_done"] == 4 and line["failed_step"] == 0
    assert line["exchange"].startswith("fused peer-memory halo") and line["value"] > 0
    assert line["gpu_launches"] > 0
    assert line["scaling"] == "strong" and 0.0 < line["roofline"]["frac"] < 1.0


def _peer_vs_single(P, mode, world, nsteps, bnd=None, src=None, linear=False):
    """Decomposed run (in-process ranks) and the single-engine run of P."""
    import torch

    ed = P.engine_desc()
    periodic = bool(ed.periodic_xi)
    sls = sharded.slabs(ed.Nxi, periodic, world)
    dev = torch.device("cuda", 0)
    E = Engine.from_problem(P, mode=mode)
    engines = [Engine(sharded.subset_desc(ed, sl), mode) for sl in sls]
    if linear:  # the full engine's row weights (gaptooth.cpp:377-394) on every slab
        w = E.set_linear()
        for Es in engines:
            Es.set_linear(w)
    runners = sharded.local_peer_group(engines, sls, ed.Neta, dev, k=ed.k)
    U0 = P.initial_field()
    Ut = torch.from_numpy(U0.reshape(-1).copy()).to(dev)
    res = sharded.run_peer(runners, [Ut] * world, nsteps, P.desc.T / P.desc.Nt, 0.0, bnd, src_table=src)
    full = assemble([r.U.cpu().numpy() for r in res], sls, P.shape, periodic)
    Uref, st = E.run(U0, nsteps, bnd=bnd, src_time=src)
    assert all(r.failed_step == 0 and r.steps_done == nsteps for r in res)
    return full, Uref


@pytest.mark.parametrize("mode", [EXACT, FAST], ids=["exact", "fast"])
def test_peer_halo_adi_with_source(mode, gpu):
    """The fused halo store in the ADI kernels (EXACT and FAST families) and the
    per-step separable-source factors (problem1, the reference's Table-1 setup)."""
    P = Problem(configs.copy_desc(configs.load("ref_table1_cdr_const")[0]))
    n = 6
    full, Uref = _peer_vs_single(P, mode, 3, n, P.boundary_table(0.0, n), P.source_time(0.0, n))
    assert np.array_equal(full, Uref)


@pytest.mark.parametrize("name", ["c1_diffusion", "c3_annulus"])
def test_peer_halo_linear_response_step(name, gpu):
    """The fused halo store in the linear-response step (k_linear_step,
    gaptooth.cpp:396-418) with the full engine's row weights on every slab."""
    P = Problem(configs.load(name)[0])
    full, Uref = _peer_vs_single(P, EXACT, 2, 15, linear=True)
    assert np.array_equal(full, Uref)


@pytest.mark.parametrize("name,over", [("c1_diffusion", {"k": 1}), ("c3_annulus", {"k": 2}),
                                       ("ref_table1_cdr_const", {"problem": abi.PD_PROBLEM_REF_CDR_VAR, "k": 1})],
                         ids=["c1-k1", "c3-k2", "adi-var-k1"])
@pytest.mark.parametrize("mode", [EXACT, FAST], ids=["exact", "fast"])
def test_peer_halo_k_substeps(name, over, mode, gpu):
    """k > 0 (cpi.cpp:58-77 chains k+1 gap-tooth substeps): each substep and the
    extrapolation store their edge columns into the neighbours' matching buffers
    (pd_gaptooth_substep_halo / pd_extrapolate_halo), k+2 counter advances per
    projective step; bit-identical to the single engine."""
    P = Problem(configs.copy_desc(configs.load(name)[0], **over))
    assert P.desc.k == over["k"]
    n = 8
    full, Uref = _peer_vs_single(P, mode, 3, n, P.boundary_table(0.0, n), P.source_time(0.0, n))
    assert np.array_equal(full, Uref)
