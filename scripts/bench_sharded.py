"""Strong scaling of the xi-slab decomposition (paper_2405_08764_b200/sharded.py) over N GPUs
with NCCL point-to-point halo columns and an all-reduce guard per macro step.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
      --master-port 29511 scripts/bench_sharded.py [--config c4_shear] [--steps 50]

Prints one JSON line (rank 0): total patch-node updates/s over the device time (max over ranks)
of `steps` macro steps, the per-rank patch counts, and the same run's single-engine reference
time when N == 1.  bench.py's contract line stays the replicas run; this is the decomposition."""
import argparse, json, os, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2405_08764_b200 import configs, sharded  # noqa: E402
from paper_2405_08764_b200.engine import Engine, Problem, _check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4_shear")
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
P = Problem(configs.load(a.config)[0])
ed = P.engine_desc()
sl = sharded.slabs(ed.Nxi, bool(ed.periodic_xi), world)[rank]
E = Engine(sharded.subset_desc(ed, sl))
stream = torch.cuda.current_stream(dev)
_check(lib().pd_engine_set_stream(E.h, stream.cuda_stream), E.h)  # engine kernels ordered with NCCL on this stream
step = sharded.device_step_fn(E, P.desc.k, E.perim, dev)
runner = sharded.ShardedRun(sl, ed.Neta, step, dist, k=P.desc.k)
U0 = torch.from_numpy(P.initial_field().reshape(-1).copy()).to(dev)
dt = P.desc.T / P.desc.Nt
runner.run(U0.clone(), a.warmup, dt)
dist.barrier()
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(stream)
U, done, failed = runner.run(U0.clone(), a.steps, dt)
ev1.record(stream)
torch.cuda.synchronize()
ms = torch.tensor([ev0.elapsed_time(ev1)], device=dev, dtype=torch.float64)
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
cnt = torch.tensor([E.P], device=dev, dtype=torch.float64)
dist.all_reduce(cnt)
n1, n2 = P.desc.nx + 1, P.desc.ny + 1
upd = ed.npatches * n1 * n2 * P.desc.nt * a.steps
line = {"metric": "FP64 patch-node micro-updates/s (xi-slab decomposition)", "value": upd / (ms.item() * 1e-3),
        "unit": "patch-node updates/s", "n_gpus": world, "steps": a.steps, "ms_per_step": ms.item() / a.steps,
        "scaling": "strong", "config": {"workload": a.config, "patches": ed.npatches, "patches_per_rank_max": E.P,
                                       "partition": f"{world} xi-slabs", "exchange": "NCCL P2P halo columns + "
                                       "all-reduce(max) guard per macro step"},
        "steps_done": done, "failed_step": failed}
assert int(cnt.item()) == ed.npatches
if rank == 0:
    print(json.dumps(line), flush=True)
dist.destroy_process_group()
