#!/usr/bin/env python
"""Benchmark of the B200 gap-tooth hot path (BASELINE.json metric).

One *step* = one projective forward-Euler macro step (k = 0: one fused
gap-tooth substep over every patch + extrapolation + boundary refresh + the
blow-up guard) of the headline workload, config 4 (512x512 patches of 16x16
micro nodes, K = 50 micro-steps, 9-point non-orthogonal CDR, FP64).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c4_shear] [--no-cpu-baseline] [--sweep]

N = 1: the device-resident single-engine loop (pd_run_device).  N > 1 is
launched by torchrun (one process per GPU): the workload is split into
xi-slabs of patch columns (sharded.py), every rank advances its own
patches and its step kernel stores its two edge columns straight into the
neighbours' field buffers (CUDA IPC mappings over NVLink/NVSwitch) and bumps
their link counters; each rank's stream waits on its own counters before the
next step (pd_projective_step_halo / pd_stream_wait_flag), with one
all-reduce(max) guard per run (--exchange nccl: NCCL point-to-point halo
columns instead) — strong scaling, value = all patches' updates /
max-over-ranks time.

--impl reference times the reference's CPU implementation of the path on this
host's cores: for the shear-cdr workloads (configs 4/5, whose mixed term the
unmodified reference rejects, microsim.cpp:239-244) the restated oracle
(oracle/pd_oracle.c) over the FULL workload every step, with inputs built by
the oracle alone (oracle/pd_oracle_problem.c — the product library is never
loaded); for configs 1-3 the unmodified reference (oracle/_ref).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np

from paper_2405_08764_b200 import abi, configs  # noqa: E402  (pure Python: no library load)

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]
UNIT = "patch-node updates/s"
PARITY_TOL = 1e-11  # north_star: FP64 macro fields within 1e-11 relative max-norm


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json"
    return 6650.0, "fallback (B200_PROFILING.md)"


def flops_per_update(mixed: bool) -> int:
    # folded 5-point = 1 mul + 4 FMA = 9 flop; 9-point adds 5 -> 14
    return 14 if mixed else 9


PERIODIC = (abi.PD_PROBLEM_ANNULUS_NONAXI, abi.PD_PROBLEM_REF_ANNULUS)


def workload(desc):
    """(patches, micro nodes per patch, micro-steps per macro step) from the
    problem description alone (gaptooth.cpp:251-280 patch list)."""
    n1, n2 = desc.nx + 1, desc.ny + 1
    i_lo = 0 if desc.problem in PERIODIC else 1
    P = (desc.N_xi - i_lo) * (desc.N_eta - 1)
    return P, n1 * n2, desc.nt * (desc.k + 1)


def bench_config(name, desc, world):
    """The `config` object, identical in both arms (ours / reference)."""
    P, N, K = workload(desc)
    mixed = desc.problem == abi.PD_PROBLEM_SHEAR_CDR
    table = P * N * 8 * (6 if mixed else 5)
    return {"workload": name, "patches": P, "micro_nodes": N, "K": K,
            "stencil": "9-point (mixed term)" if mixed else "5-point",
            "parallelism": "single GPU" if world == 1 else f"xi-slab decomposition over {world} GPUs",
            "l2": (f"inputs larger than L2: {table / 1e9:.2f} GB of folded weights streamed per macro step "
                   f"(> 126 MB L2)") if table > 126e6 else
                  (f"L2-resident: {table / 1e6:.1f} MB of weights (< 126 MB L2), no flush between steps "
                   f"(the reference re-reads the same tables every step)")}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_traffic(config_name: str):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None, None
    d = json.loads(p.read_text())
    ent = d.get(config_name)
    if not ent:
        return None, None
    return ent.get("dram_bytes_per_launch"), ent.get("source")


def single_thread_rate(O, ed, U0, P, N, K, target_s=2.0):
    """The restated oracle on ONE host core (the reference is single-threaded by
    design, gaptooth.cpp:362), bounded patch sample."""
    threads = O.threads
    O.set_threads(1)
    try:
        rng = np.random.default_rng(3)
        n = min(P, 16)
        idx = np.sort(rng.choice(P, n, replace=False)).astype(np.int32)
        _, sec = O.patch_subset(ed, U0, 0.0, idx)
        n = int(min(P, max(n, (n / max(sec, 1e-9)) * target_s)))
        idx = np.sort(rng.choice(P, n, replace=False)).astype(np.int32)
        _, sec = O.patch_subset(ed, U0, 0.0, idx)
        return n * N * K / sec, n
    finally:
        O.set_threads(threads)


def cpu_baseline(ed, U0, P, N, K, target_s=8.0):
    """The restated oracle (port) on this host's cores over a bounded patch
    sample; returns (cpu_baseline object, sample indices, oracle averages)."""
    from oracle.pyoracle import Restated  # checker / CPU baseline only

    O = Restated()
    threads = O.threads
    rng = np.random.default_rng(1)
    n = min(P, 256)
    idx = np.sort(rng.choice(P, n, replace=False)).astype(np.int32)
    _, sec = O.patch_subset(ed, U0, 0.0, idx)
    rate = n * N * K / max(sec, 1e-9)
    n2 = int(min(P, max(n, rate * target_s / (N * K))))
    idx = np.sort(rng.choice(P, n2, replace=False)).astype(np.int32)
    avg, sec = O.patch_subset(ed, U0, 0.0, idx)
    st_rate, st_n = single_thread_rate(O, ed, U0, P, N, K)
    obj = {"value": n2 * N * K / sec, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"{n2} of {P} patches, one gap-tooth substep (K={K} micro-steps each) of the "
                     f"restated oracle (oracle/pd_oracle.c, OpenMP over patches), {sec:.2f} s",
           "single_thread_value": st_rate, "single_thread_sample": f"{st_n} patches on 1 core",
           "nproc": os.cpu_count()}
    return obj, idx, avg


def patch_parity(S, ed, idx, avg):
    """max |GPU - oracle| / max |oracle| over the sampled patches' restricted
    averages after one gap-tooth substep (patch-local, test_gaptooth.cpp:244-255)."""
    pij = np.ctypeslib.as_array(ed.patch_ij, shape=(ed.npatches, 2))[idx]
    got = S[pij[:, 0], pij[:, 1]]
    return float(np.abs(got - avg).max() / max(np.abs(avg).max(), 1e-300))


# ---------------------------------------------------------------------------
# --impl reference
# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    """The reference's CPU implementation of the path on this host's cores."""
    if rank != 0:
        return 0
    desc, _ = configs.load(args.config)
    P, N, K = workload(desc)
    cfg = bench_config(args.config, desc, world)
    base = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg}
    if desc.problem == abi.PD_PROBLEM_SHEAR_CDR:
        # configs 4/5: the unmodified reference rejects b != 0 (MixedTermUnsupported,
        # microsim.cpp:239-244) -> the restated oracle (reference + mixed term), the whole
        # workload every step, inputs from the oracle's own builder
        from oracle.pyoracle import Restated

        O = Restated()
        t0 = time.perf_counter()
        r, ed, U0 = O.shear_problem(desc)
        build_s = time.perf_counter() - t0
        dt = r.T / r.Nt
        U = U0
        for n in range(args.warmup):
            st, U = O.projective_step(ed, U, n * dt)
            assert st == 0, st
        secs = []
        for n in range(args.steps):
            t1 = time.perf_counter()
            st, U = O.projective_step(ed, U, (args.warmup + n) * dt)
            secs.append(time.perf_counter() - t1)
            assert st == 0, st
        sec = sum(secs)
        value = P * N * K * args.steps / sec
        st_rate, st_n = single_thread_rate(O, ed, U0, P, N, K)
        kind, cores = "port", O.threads
        sample = (f"each step: one full projective macro step over all {P} patches of the restated oracle "
                  f"(oracle/pd_oracle.c; the reference itself rejects b != 0), OpenMP {cores} threads; "
                  f"tables built by oracle/pd_oracle_problem.c in {build_s:.1f} s (untimed)")
        extra = {"single_thread_value": st_rate, "single_thread_sample": f"{st_n} patches on 1 core",
                 "nproc": os.cpu_count()}
    else:
        from oracle.pyoracle import Reference, reference_available, ref_problem_desc

        if not reference_available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (the unmodified reference) "
                              "was not built: it needs /root/reference at build time"}), flush=True)
            return 0
        # the unmodified reference (oracle/_ref): cpi::projective_step, single-threaded by design
        ref = Reference().engine(ref_problem_desc(desc))
        rd = ref.pdesc
        U = ref.initial_field()
        for n in range(args.warmup):
            U = ref.projective_step(U, n * rd.T / rd.Nt)
        U, sec = ref.steps(U, args.warmup, args.steps)
        value = P * N * K * args.steps / sec
        kind, cores = "reference", 1
        sample = f"{args.steps} full macro steps of the unmodified reference (single-threaded by design, " \
                 f"proj/src/gaptooth.cpp:362)"
        extra = {"nproc": os.cpu_count()}
    line = dict(base, value=value, ms_per_step=1e3 * sec / args.steps,
                cpu_baseline=dict({"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
                                  **extra),
                e2e={"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# --sweep (config 5)
# ---------------------------------------------------------------------------
def run_sweep(args):
    """BASELINE config 5: updates/s and roofline fraction at every sweep point,
    next to the restated CPU oracle on a bounded patch sample (host cores), and
    the parity of the GPU's substep against that same oracle sample."""
    import gc

    import torch

    from oracle.pyoracle import Restated
    from paper_2405_08764_b200.engine import Engine, Problem, fp64_peak

    base, vals = configs.load("c5_sweep")
    sizes = [int(x) for x in vals["sweep.log2_patches"].split(",")]
    nodes_l = [int(x) for x in vals["sweep.micro_nodes"].split(",")]
    Ks = [int(x) for x in vals["sweep.K"].split(",")]
    if args.sweep_max_log2:
        sizes = [s for s in sizes if s <= args.sweep_max_log2]
    if args.sweep_nodes:
        nodes_l = [int(x) for x in args.sweep_nodes.split(",")]
    p64, ghz = fp64_peak(200.0)
    bw, bw_src = peaks()
    O = Restated()
    out_path = ROOT / "profiles" / f"c5_sweep_{args.tag}.jsonl"
    rows = []
    for nodes in nodes_l:
        for lp in sizes:
            for K in Ks:
                d = configs.sweep_desc(base, lp, nodes, K)
                t0 = time.perf_counter()
                prob = Problem(d)
                eng = Engine.from_problem(prob, mode=configs.MODE[args.mode])
                build_s = time.perf_counter() - t0
                P, N, Kk = workload(prob.desc)
                mixed = eng.mixed
                U0 = prob.initial_field()
                dU = torch.from_numpy(U0.ravel()).cuda()
                dS = torch.empty_like(dU)
                eng.run_device(dU.data_ptr(), dS.data_ptr(), 3)  # warm-up
                dU.copy_(torch.from_numpy(U0.ravel()))
                steps = max(3, min(20, int(2e11 // (P * N * K)) or 3))
                torch.cuda.synchronize()
                st = eng.run_device(dU.data_ptr(), dS.data_ptr(), steps)
                # kernel-only time: best of three 3-launch averages (one noisy sample
                # otherwise moves a point's fraction by 0.1)
                kms = min(eng.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), reps=3) for _ in range(3))
                upd = P * N * K
                flops, byts = upd * flops_per_update(mixed), P * (N * 8 * (6 if mixed else 5) + 16)
                t_fp, t_bw = flops / (p64 * 1e12), byts / (bw * 1e9)
                bound = "fp64" if t_fp >= t_bw else "hbm"
                frac = max(t_fp, t_bw) / (kms * 1e-3)
                # CPU oracle on a bounded sample (about 1 s of host work) and the
                # GPU's substep on the same patches
                ed = prob.engine_desc()
                n = min(P, max(8, int(2e7 // (N * K))))
                idx = np.sort(np.random.default_rng(lp).choice(P, n, replace=False)).astype(np.int32)
                avg, csec = O.patch_subset(ed, U0, 0.0, idx)
                par = patch_parity(eng.step_direct(U0, 0.0), ed, idx, avg)
                row = {"config": "c5_sweep", "log2_patches": lp, "patches": P, "micro_nodes": f"{nodes}x{nodes}", "K": K,
                       "kernel_family": "fast" if eng.mode == abi.PD_MODE_FAST else "exact",
                       **({} if eng.mode == abi.PD_MODE_FAST else {"exact_tile": bool(eng.exact_tile)}),
                       "updates_per_s": upd / (kms * 1e-3), "step_updates_per_s": upd * steps / (st.device_ms * 1e-3),
                       "kernel_ms": kms, "ms_per_macro_step": st.device_ms / steps, "roofline_bound": bound,
                       "roofline_frac": frac, "fp64_peak_tflops": p64, "hbm_peak_gbs": bw,
                       "achieved_tflops": flops / (kms * 1e-3) / 1e12, "achieved_gbs": byts / (kms * 1e-3) / 1e9,
                       "parity_rel": par, "parity_patches": n, "parity_ok": par < PARITY_TOL,
                       "cpu_oracle_updates_per_s": n * N * K / csec, "cpu_cores": O.threads, "cpu_sample_patches": n,
                       "host_build_s": build_s, "device_gb": eng.device_bytes / 1e9}
                rows.append(row)
                print(json.dumps(row), flush=True)
                del eng, prob, dU, dS
                gc.collect()
                torch.cuda.empty_cache()
    (ROOT / "profiles").mkdir(exist_ok=True)
    with open(out_path, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def roofline(eng, desc, kms, mixed, config_name):
    from paper_2405_08764_b200.engine import fp64_peak

    P, N, K = workload(desc)
    p64, ghz = fp64_peak(200.0)
    bw, bw_src = peaks()
    fpu = flops_per_update(mixed)
    ncoef = 6 if mixed else 5
    flops_launch = P * N * K * fpu
    bytes_launch = P * (N * 8 * ncoef + 16)
    t_fp = flops_launch / (p64 * 1e12)
    t_bw = bytes_launch / (bw * 1e9)
    # the ncu summary is per kernel: EXACT-family launches have their own entry
    traffic, traffic_src = load_traffic(config_name if eng.mode == abi.PD_MODE_FAST else config_name + "_exact")
    if t_fp >= t_bw:
        roof = {"bound": "fp64", "achieved": flops_launch / (kms * 1e-3) / 1e12, "peak": p64, "unit": "TFLOP/s"}
    else:
        roof = {"bound": "hbm", "achieved": bytes_launch / (kms * 1e-3) / 1e9, "peak": bw, "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = traffic
    roof.update({
        "kernel": ("k_fast (fused gap-tooth substep)" if eng.mode == abi.PD_MODE_FAST
                   else "k_exact_tile (EXACT, register-blocked)" if eng.exact_tile else "k_gaptooth_exact"),
        "kernel_ms": kms, "flops_per_update": fpu, "algorithmic_flops_per_launch": flops_launch,
        "algorithmic_bytes_per_launch": bytes_launch,
        "peak_source": f"FP64 DFMA microbenchmark measured in this run at {ghz:.3f} GHz; HBM {bw} GB/s from {bw_src}",
        "roofline_time_ms": max(t_fp, t_bw) * 1e3, "frac_of_roofline_time": max(t_fp, t_bw) * 1e3 / kms,
        "traffic_source": traffic_src})
    return roof


def run_single(args, desc):
    """N = 1: the device-resident macro loop of one engine (pd_run_device)."""
    import ctypes as C

    import torch

    from paper_2405_08764_b200.engine import Engine, Problem, _check
    from paper_2405_08764_b200.engine import lib as _lib

    torch.cuda.set_device(0)
    prob = Problem(desc)
    r = prob.desc
    eng = Engine.from_problem(prob)
    P, N, K = workload(r)
    ed = prob.engine_desc()
    mixed = eng.mixed
    U0 = prob.initial_field()
    NF = U0.size
    dev = torch.device("cuda", 0)
    dU = torch.from_numpy(U0.ravel()).to(dev)
    dS = torch.empty_like(dU)
    torch.cuda.synchronize()

    # warm-up (untimed), from the same initial field
    eng.run_device(dU.data_ptr(), dS.data_ptr(), args.warmup)
    dU.copy_(torch.from_numpy(U0.ravel()))
    torch.cuda.synchronize()

    # ---- timed region: exactly K macro steps, device-resident -------------
    clocks = ClockSampler(0)
    clocks.start()
    torch.cuda.synchronize()
    stats = eng.run_device(dU.data_ptr(), dS.data_ptr(), args.steps)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = stats.device_ms
    value = P * N * K * args.steps / (ms * 1e-3)

    # ---- dominant kernel + FP64 peak + roofline ----------------------------
    if int(stats.kernel_launches) == 1:
        # the whole run was ONE cooperative launch (k_fast_run: fused step + refresh +
        # guard per grid barrier): its per-macro-step share is the step itself
        kms = ms / args.steps
        roof = roofline(eng, r, kms, mixed, args.config)
        roof["kernel"] = "k_fast_run (the whole timed run in one cooperative launch; per macro step)"
        roof["kernel_share_of_step"] = 1.0
    else:
        kms = eng.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), reps=5)
        roof = roofline(eng, r, kms, mixed, args.config)
        roof["kernel_share_of_step"] = kms / (ms / args.steps)

    # ---- end to end through the host C-ABI (pd_projective_step) ------------
    ke = max(3, min(args.steps, 20))
    Uh = torch.from_numpy(U0.ravel().copy()).pin_memory()
    Oh = torch.empty_like(Uh).pin_memory()
    Uh_np, Oh_np = Uh.numpy().reshape(U0.shape), Oh.numpy().reshape(U0.shape)
    eng.projective_step(Uh_np, 0.0)  # warm
    L = _lib()
    dp = C.POINTER(C.c_double)
    dtm = r.T / r.Nt
    t0 = time.perf_counter()
    cur, nxt = Uh_np, Oh_np
    for n in range(ke):
        _check(L.pd_projective_step(eng.h, cur.ctypes.data_as(dp), nxt.ctypes.data_as(dp), n * dtm, None, None),
               eng.h)
        cur, nxt = nxt, cur
    e2e_s = time.perf_counter() - t0
    e2e = {"value": P * N * K * ke / e2e_s, "unit": UNIT, "h2d_bytes_per_step": NF * 8,
           "d2h_bytes_per_step": NF * 8, "steps": ke,
           "path": "pd_projective_step (host pinned buffers, H2D + fused kernels + D2H each step)"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": bench_config(args.config, desc, 1),
            "kernel_family": "fast" if eng.mode == abi.PD_MODE_FAST else "exact",
            "roofline": roof, "e2e": e2e, "gpu_launches": int(stats.kernel_launches), "clocks": clk}
    if not args.no_cpu_baseline:
        cb, idx, avg = cpu_baseline(ed, U0, P, N, K)
        line["cpu_baseline"] = cb
        # parity of the same launch configuration against that oracle sample
        S = eng.step_direct(U0, 0.0)
        par = patch_parity(S, ed, idx, avg)
        line["parity"] = {"rel_err": par, "patches": len(idx), "tol": PARITY_TOL, "ok": par < PARITY_TOL,
                          "check": "restricted averages of one gap-tooth substep from the initial field, "
                                   "GPU vs the restated oracle on the cpu_baseline sample"}
    print(json.dumps(line), flush=True)
    return 0


def run_sharded(args, desc, rank, world, local):
    """N > 1: xi-slab strong scaling (sharded.py).  Default exchange: the fused
    peer-memory halo (each rank's step kernel stores its edge columns into the
    neighbours' buffers over NVLink/NVSwitch through CUDA IPC mappings; the
    streams wait on link counters; no NCCL in the loop).  --exchange nccl: NCCL
    point-to-point halo columns (the baseline)."""
    import torch
    import torch.distributed as dist

    from paper_2405_08764_b200 import sharded
    from paper_2405_08764_b200.engine import Engine, Problem

    # PD_BENCH_ONE_DEVICE=1 (tests only): every rank on cuda:0 over gloo, to run
    # this code path on a one-GPU box — its timings are not scaling numbers
    one_dev = os.environ.get("PD_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if one_dev:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    prob = Problem(desc)
    r = prob.desc
    ed = prob.engine_desc()
    P, N, K = workload(r)
    sl = sharded.slabs(ed.Nxi, bool(ed.periodic_xi), world)[rank]
    eng = Engine(sharded.subset_desc(ed, sl))
    # one node, one process per GPU: the neighbour rank's device is its rank
    ndev = torch.cuda.device_count()
    peer_ok = args.exchange == "peer" and (one_dev or all(
        nb < ndev and nb != local and torch.cuda.can_device_access_peer(local, nb) for _, nb, _ in sharded.halo_links(sl)))
    if args.exchange == "nccl" and one_dev:
        raise SystemExit("--exchange nccl needs one GPU per rank")
    cdev = torch.device("cpu") if one_dev else dev  # collectives' tensors (gloo: host)
    ok = torch.tensor([1.0 if peer_ok else 0.0], device=cdev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    use_peer = bool(ok.item())
    dt = r.T / r.Nt
    U0 = torch.from_numpy(prob.initial_field().reshape(-1).copy()).to(dev)
    run = None
    if use_peer:
        # the IPC mappings are the one step that can fail on a node (no P2P path):
        # agree across ranks and fall back to the NCCL exchange rather than abort
        try:
            run = sharded.peer_runner(eng, sl, ed.Neta, dist, dev, k=ed.k)
            ok_ipc = 1.0
        except Exception as x:  # noqa: BLE001 - reported, then the NCCL transport runs
            print(f"rank {rank}: peer-memory halo unavailable ({x}); using NCCL", file=sys.stderr, flush=True)
            ok_ipc = 0.0
        flag = torch.tensor([ok_ipc], device=cdev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if flag.item() < 1.0:
            if run is not None:
                sharded.close_peer_runner(run)
            run, use_peer = None, False
    if use_peer:

        def red(x):
            t = x.detach().to(cdev).clone()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t.cpu()

        def go(U, n, t0=0.0):
            return sharded.run_peer([run], [U], n, dt, t0, reduce_max=red, barrier=dist.barrier)[0]
        exchange = ("fused peer-memory halo: the step kernel stores its edge columns into the neighbours' field "
                    "buffers (CUDA IPC over NVLink/NVSwitch) and bumps their link counters; streams wait on "
                    "counters (cuStreamWaitValue32); one all-reduce(max) guard per run")
    else:
        runner = sharded.device_runner(eng, sl, ed, dist, dev)

        def go(U, n, t0=0.0):
            return runner.run_deferred(U, n, dt, t0)
        exchange = ("NCCL point-to-point halo columns (one macro column per neighbour per step) + "
                    "device all-reduce(max) guard, on the engine's stream")
    go(U0.clone(), args.warmup)
    dist.barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    U = U0.clone()
    l0 = eng.launch_count
    dist.barrier()
    torch.cuda.synchronize()
    res = go(U, args.steps)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = eng.launch_count - l0
    t = torch.tensor([res.device_ms], device=cdev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = P * N * K * args.steps / (ms * 1e-3)

    # e2e: host field in (pinned) -> sharded step -> host field out, every step
    ke = max(3, min(args.steps, 20))
    Uh = torch.from_numpy(prob.initial_field().reshape(-1).copy()).pin_memory()
    dist.barrier()
    t0 = time.perf_counter()
    for n in range(ke):
        Ud = Uh.to(dev, non_blocking=True)
        Ud = go(Ud, 1, n * dt).U
        Uh.copy_(Ud)
    torch.cuda.synchronize()
    e2e_s = torch.tensor([time.perf_counter() - t0], device=cdev, dtype=torch.float64)
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    NF = Uh.numel()
    e2e = {"value": P * N * K * ke / float(e2e_s.item()), "unit": UNIT, "h2d_bytes_per_step": NF * 8,
           "d2h_bytes_per_step": NF * 8, "steps": ke,
           "path": "host field (pinned) -> per-rank slab step + halo exchange -> host, each step"}
    mine = torch.tensor([eng.P], device=cdev, dtype=torch.float64)
    most = mine.clone()
    dist.all_reduce(most, op=dist.ReduceOp.MAX)
    roof = None
    if rank == 0:
        # roofline of the busiest rank's slab: its patches' algorithmic flops / bytes per macro
        # step against the whole step's device time (the step kernel is > 99 % of it at N = 1)
        from paper_2405_08764_b200.engine import fp64_peak
        p64, ghz = fp64_peak(200.0)
        bw, bw_src = peaks()
        mixed = bool(eng.mixed)
        Pm = int(most.item())
        t_fp = Pm * N * K * flops_per_update(mixed) / (p64 * 1e12)
        t_bw = Pm * (N * 8 * (6 if mixed else 5) + 16) / (bw * 1e9)
        step_s = ms * 1e-3 / args.steps
        roof = {"bound": "fp64" if t_fp >= t_bw else "hbm",
                "achieved": (Pm * N * K * flops_per_update(mixed) / step_s / 1e12 if t_fp >= t_bw
                             else Pm * (N * 8 * (6 if mixed else 5) + 16) / step_s / 1e9),
                "peak": p64 if t_fp >= t_bw else bw, "unit": "TFLOP/s" if t_fp >= t_bw else "GB/s",
                "frac": max(t_fp, t_bw) / step_s, "traffic": None,
                "kernel": "per-rank fused step over the busiest slab (whole macro step timed, max over ranks)",
                "peak_source": f"FP64 DFMA microbenchmark on rank 0 at {ghz:.3f} GHz; HBM {bw} GB/s from {bw_src}"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": bench_config(args.config, desc, world),
                "kernel_family": "fast" if eng.mode == abi.PD_MODE_FAST else "exact",
                "patches_per_rank_max": int(most.item()), "steps_done": res.steps_done,
                "failed_step": res.failed_step, "exchange": exchange,
                **({"one_device_test": "all ranks on cuda:0 (PD_BENCH_ONE_DEVICE): not a scaling number"}
                   if one_dev else {}),
                "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk}
        print(json.dumps(line), flush=True)
    if use_peer:
        dist.barrier()
        sharded.close_peer_runner(run)
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4_shear")
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="config-5 sweep -> profiles/c5_sweep_<tag>.jsonl")
    ap.add_argument("--sweep-max-log2", type=int, default=0)
    ap.add_argument("--sweep-nodes", default="")
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N > 1: fused peer-memory halo (default) or NCCL point-to-point halo columns")
    args = ap.parse_args()
    if args.sweep:
        return run_sweep(args)
    if args.warmup < 3:
        args.warmup = 3

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    desc, _ = configs.load(args.config)
    desc.mode = configs.MODE[args.mode]
    if world == 1:
        return run_single(args, desc)
    return run_sharded(args, desc, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
