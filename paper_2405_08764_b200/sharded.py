"""Multi-process slab decomposition of the macro loop.

Within one gap-tooth substep the patches are independent; across substeps each
patch needs its 3x3 macro stencil (gaptooth.cpp:74-104).  So the patch columns
i in [i_lo, Nxi-1] are split into contiguous xi-slabs, one per rank; every rank
keeps a full-size macro field buffer but only its own columns (plus one halo
column on each side, and the global boundary) are ever current.  Per substep:

  1. the rank's engine advances its own patches (the fused device step);
  2. the two edge columns go to the neighbouring ranks and the two halo columns
     come back (one macro column = Neta+1 contiguous doubles in the i-major
     Field2D layout, field.hpp:20-27; periodic xi wraps rank 0 <-> rank N-1);
  3. the blow-up guard (cpi.cpp:187-202) reduces max |U| over ranks (one
     all-reduce of a single double).

Results do not depend on the decomposition: every patch value is computed from
the same stencil values in the same arithmetic, so the sharded run equals the
single-engine run bit for bit (tests/test_dist.py, tests/test_gpu_peer.py).

Two transports:

* ``PeerRun`` / ``run_peer`` (the product path, bench.py --gpus N): step 2 is
  fused into step 1 — the step kernel stores its edge columns straight into the
  neighbours' buffers (NVLink peer / CUDA IPC mappings) and bumps their link
  counters, each rank's stream waits on its own counters (stream memory
  operations), and the guard is ONE all-reduce of the per-step maxima after the
  loop;
* ``ShardedRun`` (the baseline, and the CPU tests): torch.distributed
  point-to-point ops for step 2 — NCCL on GPUs, gloo on CPU; the compute is
  injected (``step_fn``: the engine's fused projective step on device buffers,
  or the restated oracle in the CPU tests).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import abi
from .abi import EngineDesc, perimeter_len


@dataclass
class Slab:
    rank: int
    world: int
    i0: int  # first owned patch column
    i1: int  # one past the last owned patch column
    periodic: bool
    Nxi: int

    def left(self) -> int | None:
        """Rank owning column i0-1 (None: the global boundary)."""
        if self.rank > 0:
            return self.rank - 1
        return self.world - 1 if self.periodic and self.world > 1 else None

    def right(self) -> int | None:
        if self.rank < self.world - 1:
            return self.rank + 1
        return 0 if self.periodic and self.world > 1 else None


def slabs(Nxi: int, periodic: bool, world: int) -> list[Slab]:
    """Contiguous, balanced xi-slabs of the patch columns (gaptooth.cpp:251-280)."""
    i_lo, i_hi = (0 if periodic else 1), Nxi - 1
    ncol = i_hi - i_lo + 1
    if world > ncol:
        raise ValueError(f"{world} ranks for {ncol} patch columns")
    out, start = [], i_lo
    for r in range(world):
        n = ncol // world + (1 if r < ncol % world else 0)
        out.append(Slab(r, world, start, start + n, periodic, Nxi))
        start += n
    return out


def subset_desc(ed: EngineDesc, slab: Slab) -> EngineDesc:
    """pd_engine_desc restricted to the slab's patches (reference order kept),
    with only the coefficient sets those patches use."""
    if not ed.coeffs:
        raise ValueError("subset_desc slices host coefficient tables (build the problem with coeff_gen=PD_COEFF_HOST)")
    P = ed.npatches
    pij = np.ctypeslib.as_array(ed.patch_ij, shape=(P, 2)).copy()
    sel = np.nonzero((pij[:, 0] >= slab.i0) & (pij[:, 0] < slab.i1))[0]
    cset = np.ctypeslib.as_array(ed.coeff_set, shape=(P,)).copy() if ed.coeff_set else np.arange(P, dtype=np.int32)
    used, remap = np.unique(cset[sel], return_inverse=True)
    n1, n2 = ed.nx + 1, ed.ny + 1
    per_set = abi.PD_NCOEF * n1 * n2
    coeffs = np.ctypeslib.as_array(ed.coeffs, shape=(ed.ncoeff_sets * per_set,))
    sub_coef = np.ascontiguousarray(coeffs.reshape(ed.ncoeff_sets, per_set)[used])
    sub_pij = np.ascontiguousarray(pij[sel].astype(np.int32))
    sub_cset = np.ascontiguousarray(remap.astype(np.int32))
    d = EngineDesc()
    for f, _ in EngineDesc._fields_:
        setattr(d, f, getattr(ed, f))
    d.npatches = len(sel)
    d.patch_ij = sub_pij.ctypes.data_as(abi._ip)
    d.ncoeff_sets = len(used)
    d.coeff_set = sub_cset.ctypes.data_as(abi._ip)
    d.coeffs = sub_coef.ctypes.data_as(abi._dp)
    if ed.source_kind == abi.PD_SOURCE_SEPARABLE and ed.source_spatial:
        sp = np.ctypeslib.as_array(ed.source_spatial, shape=(ed.ncoeff_sets * n1 * n2,))
        sub_sp = np.ascontiguousarray(sp.reshape(ed.ncoeff_sets, n1 * n2)[used])
        d.source_spatial = sub_sp.ctypes.data_as(abi._dp)
        d._keep_sp = sub_sp
    d._keep = (sub_pij, sub_cset, sub_coef, ed)
    return d


@dataclass
class RunResult:
    U: object            # this rank's full-size field after the last completed step
    steps_done: int
    failed_step: int     # 0, or the macro step whose guard tripped (cpi.cpp:187-202)
    device_ms: float     # CUDA-event time of the loop (0 on CPU)


class ShardedRun:
    """The cpi::run macro loop (cpi.cpp:175-202) over xi-slabs.

    step_fn(U_in, U_out, t, bnd) -> None advances the rank's own patches by one
    projective step (k+1 substeps + extrapolation + boundary refresh) on
    full-size field buffers (numpy arrays or torch tensors, 1-D, length NF).
    """

    def __init__(self, slab: Slab, Neta: int, step_fn, dist, group=None, stage_cpu: bool = False, k: int = 0):
        if k != 0:
            # k > 0 chains substeps inside one projective step; their halo
            # columns would have to be exchanged after every substep
            raise NotImplementedError("the xi-slab runner exchanges halos once per projective step (k = 0 only)")
        self.s = slab
        self.n2 = Neta + 1
        self.step_fn = step_fn
        self.dist = dist
        self.group = group
        self.stage_cpu = stage_cpu  # device buffers over a CPU-only transport (gloo): copy columns through the host

    def _col(self, U, i):
        return U[i * self.n2:(i + 1) * self.n2]

    def exchange(self, U):
        """Own edge columns out, halo columns in.  Per neighbour pair the
        messages are ordered (rightward first, then leftward) on both sides,
        so the exchange is unambiguous even when left == right (2 ranks,
        periodic) and with NCCL, whose point-to-point ops carry no tags."""
        import torch

        s, d = self.s, self.dist
        Nxi = s.Nxi
        left, right = s.left(), s.right()
        ops, recv = [], []
        stage = (lambda x: x.cpu()) if self.stage_cpu else (lambda x: x.contiguous())
        if right is not None:  # my last column is my right neighbour's left halo
            ops.append(d.P2POp(d.isend, stage(self._col(U, s.i1 - 1)), right, self.group))
        if left is not None:  # my first column is my left neighbour's right halo
            ops.append(d.P2POp(d.isend, stage(self._col(U, s.i0)), left, self.group))
        if left is not None:
            buf = stage(torch.empty_like(self._col(U, s.i0)))
            ops.append(d.P2POp(d.irecv, buf, left, self.group))
            recv.append(((s.i0 - 1) % Nxi if s.periodic else s.i0 - 1, buf))
        if right is not None:
            buf = stage(torch.empty_like(self._col(U, s.i0)))
            ops.append(d.P2POp(d.irecv, buf, right, self.group))
            recv.append((s.i1 % Nxi if s.periodic else s.i1, buf))
        if ops:
            for r in d.batch_isend_irecv(ops):
                r.wait()
        for i, buf in recv:
            buf = buf.to(U.device)
            U[i * self.n2:(i + 1) * self.n2] = buf
            if s.periodic and i == 0:  # the seam column mirrors column 0
                U[s.Nxi * self.n2:(s.Nxi + 1) * self.n2] = buf

    def owned_max(self, U):
        """max |U| over the rank's patch columns and the global boundary: over
        all ranks this covers every node once (the guard's scope, cpi.cpp:187-202)."""
        import torch

        s = self.s
        V = U.view(-1, self.n2)
        parts = [V[s.i0:s.i1].abs().max(), V[:, 0].abs().max(), V[:, -1].abs().max()]
        if not s.periodic:  # W/E boundary columns (periodic: column 0 is a patch column, Nxi its seam copy)
            parts += [V[0].abs().max(), V[-1].abs().max()]
        return torch.stack(parts).max()

    def run(self, U, nsteps: int, dt: float, t0: float = 0.0, bnd_table=None):
        """U: this rank's full-size field (halo columns current).  Returns
        (U, steps_done, failed_step) with cpi.cpp:187-202's guard over all ranks."""
        import torch

        d = self.dist
        red = (lambda x: x.cpu()) if self.stage_cpu else (lambda x: x)
        m0 = red(self.owned_max(U).reshape(1).clone())
        d.all_reduce(m0, op=d.ReduceOp.MAX, group=self.group)
        blowup = 10.0 * max(float(m0.item()), 1e-12)
        nxt = U.clone()  # columns a rank never computes stay finite
        for n in range(nsteps):
            self.step_fn(U, nxt, t0 + n * dt, None if bnd_table is None else bnd_table[n])
            self.exchange(nxt)
            m = red(self.owned_max(nxt).reshape(1).clone())
            d.all_reduce(m, op=d.ReduceOp.MAX, group=self.group)
            U, nxt = nxt, U
            mv = float(m.item())
            if not np.isfinite(mv) or mv > blowup:
                return U, n, n + 1
        return U, nsteps, 0

    def owned_mask(self, device=None):
        """The nodes this rank's guard covers (owned_max's scope), as a mask."""
        import torch

        s = self.s
        m = torch.zeros(s.Nxi + 1, self.n2, dtype=torch.bool, device=device)
        m[s.i0:s.i1] = True
        m[:, 0] = m[:, -1] = True
        if not s.periodic:
            m[0] = m[-1] = True
        return m.reshape(-1)

    def run_deferred(self, U, nsteps: int, dt: float, t0: float = 0.0, bnd_table=None) -> "RunResult":
        """The macro loop without any host round trip or collective per step:
        each step's owned max |U| (non-finite -> +inf) goes to a device array,
        and ONE all-reduce(max) of that array after the loop takes cpi::run's
        guard decision (cpi.cpp:187-202) for every step at once.  On a trip at
        step n the loop is replayed with the per-step guard (run()), so the
        result is run()'s: the same failing step and field.  Device time
        (CUDA events on the current stream) covers the loop and the reduction."""
        import torch

        d = self.dist
        dev = U.device
        cuda = dev.type == "cuda"
        red = (lambda x: x.cpu()) if self.stage_cpu else (lambda x: x)
        back = (lambda x: x.to(dev)) if self.stage_cpu else (lambda x: x)
        mask = self.owned_mask(dev)
        zero = torch.zeros((), dtype=U.dtype, device=dev)
        inf = torch.full((), float("inf"), dtype=U.dtype, device=dev)
        U0 = U.clone()
        if cuda:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
        m0 = red(torch.where(mask, U.abs(), zero).amax().reshape(1))
        d.all_reduce(m0, op=d.ReduceOp.MAX, group=self.group)
        blowup = 10.0 * torch.clamp(back(m0), min=1e-12)
        maxes = torch.zeros(max(nsteps, 1), dtype=U.dtype, device=dev)
        nxt = U.clone()  # columns a rank never computes stay finite
        for n in range(nsteps):
            self.step_fn(U, nxt, t0 + n * dt, None if bnd_table is None else bnd_table[n])
            self.exchange(nxt)
            m = torch.where(mask, nxt.abs(), zero).amax()
            maxes[n] = torch.where(torch.isfinite(m), m, inf)
            U, nxt = nxt, U
        allm = red(maxes)
        d.all_reduce(allm, op=d.ReduceOp.MAX, group=self.group)
        trips = back(allm)[:nsteps] > blowup
        if cuda:
            ev1.record()
        trips = trips.cpu().numpy()
        ms = 0.0
        if cuda:
            ev1.synchronize()
            ms = ev0.elapsed_time(ev1)
        if not trips.any():
            return RunResult(U, nsteps, 0, ms)
        # replay with the per-step guard: stops at the same step with the same
        # field as run() (the state right after the failing step)
        U, done, fail = self.run(U0, nsteps, dt, t0, bnd_table)
        assert fail == int(np.argmax(trips)) + 1, (fail, trips)
        return RunResult(U, done, fail, ms)

    def gather(self, U):
        """Assemble the full field on every rank from each rank's own columns."""
        import torch

        d, s = self.dist, self.s
        V = U.view(-1, self.n2)
        mine = torch.zeros(s.Nxi + 1, dtype=torch.bool, device=U.device)
        mine[s.i0:s.i1] = True
        part = torch.where(mine[:, None], V, torch.zeros_like(V))
        if self.stage_cpu:
            part = part.cpu()
        d.all_reduce(part, op=d.ReduceOp.SUM, group=self.group)
        part = part.to(U.device)
        owned = torch.zeros_like(mine)
        for sl in slabs(s.Nxi, s.periodic, s.world):
            owned[sl.i0:sl.i1] = True
        out = torch.where(owned[:, None], part, V)  # boundary columns are identical on every rank
        if s.periodic:
            out[s.Nxi] = out[0]
        return out.reshape(-1)


def device_step_fn(engine, k: int, perim: int, device):
    """The product step: the engine's fused projective step on device buffers
    (pd_projective_step_device); the boundary table row is uploaded per step."""
    import torch

    def step(U_in, U_out, t, bnd):
        b = None
        if bnd is not None:
            b = torch.as_tensor(np.ascontiguousarray(bnd).reshape(-1), device=device)
        from .engine import _check, lib

        _check(lib().pd_projective_step_device(engine.h, U_in.data_ptr(), U_out.data_ptr(), t,
                                               None if b is None else b.data_ptr(), None), engine.h)

    return step


def device_runner(engine, slab: Slab, ed: EngineDesc, dist, device, group=None) -> ShardedRun:
    """The product wiring for one rank: the slab's subset engine on the current
    torch stream (so its kernels, NCCL's halo exchange and the guard reductions
    are ordered on one stream with no host synchronisation), the fused
    projective step per macro step (pd_projective_step_device)."""
    import torch

    from .engine import _check, lib

    stream = torch.cuda.current_stream(device)
    _check(lib().pd_engine_set_stream(engine.h, stream.cuda_stream), engine.h)
    step = device_step_fn(engine, ed.k, engine.perim, device)
    return ShardedRun(slab, ed.Neta, step, dist, group=group, k=ed.k)


# ---------------------------------------------------------------------------
# Fused peer-memory halo exchange (pd_projective_step_halo):
# the step kernel of each rank stores its edge columns straight into the
# neighbours' field buffers (NVLink peer / CUDA IPC mappings) and bumps their
# link counters; each rank's stream waits on its own counters (stream memory
# operations) before the next step.  No NCCL, no host round trip per step.
# ---------------------------------------------------------------------------
FROM_LEFT, FROM_RIGHT = 0, 1  # a rank's two incoming link counters


def halo_links(slab: Slab):
    """Outgoing links of a rank: (column, neighbour rank, the neighbour's
    counter side).  My last column is my right neighbour's left halo; my first
    column is my left neighbour's right halo (gaptooth.cpp:74-104's 3x3
    stencil reads one column on each side; periodic xi wraps)."""
    out = []
    if slab.right() is not None:
        out.append((slab.i1 - 1, slab.right(), FROM_LEFT))
    if slab.left() is not None:
        out.append((slab.i0, slab.left(), FROM_RIGHT))
    return out


def incoming_sides(slab: Slab):
    """Counters this rank waits on before each step."""
    return [s for s, nb in ((FROM_LEFT, slab.left()), (FROM_RIGHT, slab.right())) if nb is not None]


class _DevArray:
    """A raw device allocation seen by torch (__cuda_array_interface__ v3)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _as_tensor(ptr: int, n: int, typestr: str, device):
    import torch

    return torch.as_tensor(_DevArray(ptr, n, typestr), device=device)


class PeerRun:
    """One rank of the cpi::run macro loop (cpi.cpp:175-202) over xi-slabs with
    the fused peer-memory halo.  X[0], X[1]: this rank's ping-pong field
    buffers; chain: k+1 substep buffers when k > 0 (cpi.cpp:58-77 chains the
    gap-tooth substeps); flags: its two incoming link counters (uint32);
    peers[rank] = (X0 ptr, X1 ptr, flags ptr, chain ptrs) of every neighbour.
    k = 0: one fused kernel per projective step (one counter advance per
    step); k > 0: k+1 substeps and the extrapolation, each storing its edge
    columns into the neighbours' matching buffer (k+2 advances per step)."""

    def __init__(self, engine, slab: Slab, Neta: int, X, flags, peers, stream, mask, k: int = 0, chain=()):
        self.e = engine
        self.s = slab
        self.n2 = Neta + 1
        self.npc = Neta - 1  # patches per column: one counter increment each per piece
        self.k = k
        self.inc = 1 if k == 0 else k + 2  # counter advances per projective step
        self.X = X
        self.chain = list(chain)
        if k > 0 and len(self.chain) != k + 1:
            raise ValueError("k > 0 needs k+1 substep buffers")
        self.flags = flags
        self.stream = stream
        self.mask = mask
        self.steps_total = 0  # counters are cumulative over the runner's life
        self.links = []
        for col, nb, side in halo_links(slab):
            x0, x1, fl, ch = peers[nb]
            self.links.append((col, (x0, x1), fl + 4 * side, tuple(ch)))
        self.sides = incoming_sides(slab)
        from .engine import _check, lib

        _check(lib().pd_engine_set_stream(engine.h, stream.cuda_stream), engine.h)

    def begin(self, U0):
        """Load the run's initial field into both buffers (stream-ordered after
        whatever produced U0 on the caller's current stream, e.g. an async H2D)."""
        import torch

        self.stream.wait_stream(torch.cuda.current_stream(self.X[0].device))
        with torch.cuda.stream(self.stream):
            self.X[0].copy_(U0)
            self.X[1].copy_(U0)
            for c in self.chain:  # columns a rank never computes stay finite
                c.copy_(U0)

    def _halo(self, dst_of):
        from . import abi

        halo = abi.HaloOut()
        halo.nlinks = len(self.links)
        for l, (col, xs, fl, ch) in enumerate(self.links):
            halo.column[l] = col
            halo.dst[l] = dst_of(xs, ch)
            halo.flag[l] = fl
        return halo

    def _wait(self, piece: int):
        """Before piece q of the run: both neighbours have finished piece q-1."""
        from .engine import _check, lib

        if piece <= 0:
            return
        target = (piece * self.npc) & 0xFFFFFFFF
        for side in self.sides:
            _check(lib().pd_stream_wait_flag(self.e.h, self.flags.data_ptr() + 4 * side, target), self.e.h)

    def enqueue_step(self, n: int, t: float, bnd, maxes, src=None):
        """Step n of the current run, all pieces at once (one rank per process)."""
        keep = None
        for keep in self.step_pieces(n, t, bnd, maxes, src):
            pass
        return keep

    def step_pieces(self, n: int, t: float, bnd, maxes, src=None):
        """Step n of the current run as a generator, one piece per next(): wait for
        both neighbours' previous piece, then the fused step (k = 0) or one of its
        k+2 pieces (own patches + edge columns into the neighbours' buffers +
        counter bumps, boundary refresh); the last piece also records this rank's
        max |U| into maxes[n].  Ranks sharing a process are advanced piece by
        piece in turn, so every stream wait is enqueued after the work it waits
        for (streams may share a hardware queue: a wait ahead of that work in the
        same queue would never be satisfied)."""
        import torch

        from .engine import _check, lib

        L, h = lib(), self.e.h
        dev = self.X[0].device
        out = (n + 1) % 2
        b = g = None
        with torch.cuda.stream(self.stream):
            if bnd is not None:  # [k+2][perimeter] refresh values of this step
                b = torch.as_tensor(np.ascontiguousarray(bnd).reshape(-1)).to(dev, non_blocking=True)
            if src is not None:  # [k+1][nt] separable-source time factors of this step
                g = torch.as_tensor(np.ascontiguousarray(src).reshape(-1)).to(dev, non_blocking=True)
        ptr = lambda x, off=0: None if x is None else x.data_ptr() + 8 * off  # noqa: E731
        first = (self.steps_total + n) * self.inc
        if self.k == 0:
            self._wait(first)
            halo = self._halo(lambda xs, ch: xs[out])
            _check(L.pd_projective_step_halo(h, self.X[n % 2].data_ptr(), self.X[out].data_ptr(), t, ptr(b), ptr(g),
                                             C.byref(halo)), h)
        else:
            perim = perimeter_len(self.s.Nxi, self.n2 - 1)
            nt = 0 if g is None else g.numel() // (self.k + 1)
            for m in range(self.k + 1):
                self._wait(first + m)
                src_buf = self.X[n % 2] if m == 0 else self.chain[m - 1]
                halo = self._halo(lambda xs, ch, m=m: ch[m])
                _check(L.pd_gaptooth_substep_halo(h, src_buf.data_ptr(), self.chain[m].data_ptr(), m,
                                                  ptr(b, perim * m), ptr(g, nt * m), C.byref(halo)), h)
                yield b, g
            halo = self._halo(lambda xs, ch: xs[out])
            _check(L.pd_extrapolate_halo(h, self.X[n % 2].data_ptr(), self.chain[self.k - 1].data_ptr(),
                                         self.chain[self.k].data_ptr(), self.X[out].data_ptr(),
                                         ptr(b, perim * (self.k + 1)), C.byref(halo)), h)
        with torch.cuda.stream(self.stream):
            mx = torch.where(self.mask, self.X[out].abs(), torch.zeros((), dtype=torch.float64, device=dev)).amax()
            maxes[n] = torch.where(torch.isfinite(mx), mx, torch.full_like(mx, float("inf")))
        yield b, g

    def result(self, nsteps: int):
        return self.X[nsteps % 2]


def _peer_guard(U0, mask, reduce_max):
    import torch

    m0 = torch.where(mask, U0.abs(), torch.zeros((), dtype=U0.dtype, device=U0.device)).amax().reshape(1)
    return 10.0 * max(float(reduce_max(m0).max().item()), 1e-12)  # cpi.cpp:142-144


def run_peer(runners, U0s, nsteps: int, dt: float, t0: float = 0.0, bnd_table=None, reduce_max=None,
             barrier=None, src_table=None) -> list[RunResult]:
    """Drive the ranks in `runners` (all ranks of an in-process group, or this
    process's one rank with torch.distributed hooks) through nsteps projective
    steps.  The guard (cpi.cpp:187-202) is taken after the loop from the
    per-step maxima (one reduction), as ShardedRun.run_deferred; on a trip the
    run is replayed up to the failing step, so the field is the one after it."""
    import torch

    reduce_max = reduce_max or (lambda x: x)
    barrier = barrier or (lambda: None)
    blowup = _peer_guard(torch.stack([U0.reshape(-1) for U0 in U0s]).reshape(-1) if len(U0s) > 1 else U0s[0],
                         torch.cat([r.mask for r in runners]) if len(runners) > 1 else runners[0].mask, reduce_max)

    def loop(steps):
        for r, U0 in zip(runners, U0s):
            r.begin(U0)
        for r in runners:
            r.stream.synchronize()
        barrier()  # every buffer holds U0 before any neighbour stores into it
        maxes = [torch.zeros(max(steps, 1), dtype=torch.float64, device=r.X[0].device) for r in runners]
        evs = []
        for r in runners:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(r.stream)
            evs.append(ev)
        keep = []
        for n in range(steps):
            gens = [r.step_pieces(n, t0 + n * dt, None if bnd_table is None else bnd_table[n], mx,
                                  None if src_table is None else src_table[n]) for r, mx in zip(runners, maxes)]
            while gens:  # piece q of every rank before piece q+1 of any (dependency order)
                live = []
                for gen in gens:
                    try:
                        keep.append(next(gen))
                        live.append(gen)
                    except StopIteration:
                        pass
                gens = live
        for r, ev in zip(runners, evs):
            ev[1].record(r.stream)
        # bounded wait: a counter that never arrives (a peer that died, a broken
        # mapping) would leave a stream waiting forever; fail loudly instead
        deadline = time.monotonic() + max(120.0, 0.5 * steps)
        for r, ev in zip(runners, evs):
            while not ev[1].query():
                if time.monotonic() > deadline:
                    raise RuntimeError(f"rank {r.s.rank}: peer halo exchange stalled (link counters not reached)")
                time.sleep(2e-5)
            r.stream.synchronize()
            r.steps_total += steps
        barrier()  # no neighbour still stores into these buffers
        ms = [ev[0].elapsed_time(ev[1]) for ev in evs]
        allm = reduce_max(torch.stack(maxes).amax(dim=0).cpu() if len(runners) > 1 else maxes[0].cpu())
        return allm[:steps].numpy(), ms

    allm, ms = loop(nsteps)
    trips = allm > blowup
    if not trips.any():
        return [RunResult(r.result(nsteps), nsteps, 0, t) for r, t in zip(runners, ms)]
    fail = int(np.argmax(trips)) + 1
    loop(fail)  # the field right after the failing step, as the per-step guard leaves it
    return [RunResult(r.result(fail), fail - 1, fail, t) for r, t in zip(runners, ms)]


def local_peer_group(engines, slab_list, Neta: int, device, k: int = 0):
    """All ranks of a decomposition in ONE process (one device or several with
    peer access): each rank's buffers and counters are plain device
    allocations, the neighbours' pointers are used directly."""
    import torch

    NF = (slab_list[0].Nxi + 1) * (Neta + 1)
    nch = k + 1 if k > 0 else 0
    bufs = [[torch.empty(NF, dtype=torch.float64, device=device) for _ in range(2)] for _ in slab_list]
    chains = [[torch.empty(NF, dtype=torch.float64, device=device) for _ in range(nch)] for _ in slab_list]
    flags = [torch.zeros(2, dtype=torch.int32, device=device) for _ in slab_list]
    peers = {r: (bufs[r][0].data_ptr(), bufs[r][1].data_ptr(), flags[r].data_ptr(),
                 tuple(c.data_ptr() for c in chains[r])) for r in range(len(slab_list))}
    out = []
    for r, (E, sl) in enumerate(zip(engines, slab_list)):
        mask = ShardedRun(sl, Neta, None, None).owned_mask(device)
        out.append(PeerRun(E, sl, Neta, bufs[r], flags[r], peers, torch.cuda.Stream(device), mask, k, chains[r]))
    return out


def peer_runner(engine, slab: Slab, Neta: int, dist, device, group=None, k: int = 0):
    """This process's rank of a one-process-per-GPU decomposition: buffers and
    counters from pd_ipc_alloc, the neighbours' opened with CUDA IPC (lazy
    peer access: NVLink/NVSwitch stores on a B200 node)."""
    import torch

    from .engine import _check, lib

    L = lib()
    NF = (slab.Nxi + 1) * (Neta + 1)

    def alloc(nbytes):
        p, h = C.c_void_p(), C.create_string_buffer(64)
        _check(L.pd_ipc_alloc(nbytes, C.byref(p), h))
        return p.value, h.raw

    (x0, h0), (x1, h1), (fl, hf) = alloc(NF * 8), alloc(NF * 8), alloc(64)
    ch = [alloc(NF * 8) for _ in range(k + 1 if k > 0 else 0)]
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, (slab.rank, h0, h1, hf, [hc for _, hc in ch]), group=group)
    peers, opened = {}, []

    def open_(hnd):
        p = C.c_void_p()
        _check(L.pd_ipc_open(C.create_string_buffer(hnd, 64), C.byref(p)))
        opened.append(p.value)
        return p.value

    for rank, a, b, f, hcs in handles:
        if rank == slab.rank:
            peers[rank] = (x0, x1, fl, tuple(pc for pc, _ in ch))
            continue
        if rank not in {nb for _, nb, _ in halo_links(slab)}:
            continue
        peers[rank] = (open_(a), open_(b), open_(f), tuple(open_(hc) for hc in hcs))
    X = [_as_tensor(x0, NF, "<f8", device), _as_tensor(x1, NF, "<f8", device)]
    chain = [_as_tensor(pc, NF, "<f8", device) for pc, _ in ch]
    flags = _as_tensor(fl, 2, "<i4", device)
    mask = ShardedRun(slab, Neta, None, None).owned_mask(device)
    run = PeerRun(engine, slab, Neta, X, flags, peers, torch.cuda.Stream(device), mask, k, chain)
    run._owned = (x0, x1, fl) + tuple(pc for pc, _ in ch)
    run._opened = opened
    return run


def close_peer_runner(run):
    """Unmap the neighbours' buffers and free this rank's (after a barrier)."""
    from .engine import lib

    L = lib()
    for p in getattr(run, "_opened", []):
        L.pd_ipc_close(C.c_void_p(p))
    for p in getattr(run, "_owned", ()):
        L.pd_device_free(C.c_void_p(p))
    run._opened, run._owned = [], ()
