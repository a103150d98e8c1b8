"""A/B of the single-launch run's synchronisation (PD_RUN_SYNC=barrier: one grid
barrier per macro step, k_fast_run; default: dataflow flags, k_fast_flow):
device ms per macro step on configs 1-3 and the small config-5 points (dev tool)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_08764_b200 import configs  # noqa: E402
from paper_2405_08764_b200.engine import Engine, Problem  # noqa: E402

mode = os.environ.get("PD_RUN_SYNC", "flow")
cases = [(n, configs.load(n)[0]) for n in ("c1_diffusion", "c2_cdr_tanh", "c3_annulus")]
base, _ = configs.load("c5_sweep")
for lp, nodes, K in [(12, 8, 10), (12, 16, 10), (13, 8, 10), (12, 8, 50), (14, 8, 10), (12, 16, 50)]:
    cases.append((f"c5-2^{lp}-{nodes}-K{K}", configs.sweep_desc(base, lp, nodes, K)))
for name, d in cases:
    P = Problem(d)
    E = Engine.from_problem(P)
    n = 200
    U0 = P.initial_field()
    b = P.boundary_table(0.0, n)
    best = 1e9
    for _ in range(3):
        U, st = E.run(U0, n, bnd=b)
        best = min(best, st.device_ms / n)
    print(f"{mode:8s} {name:22s} {1e3 * best:8.2f} us/step launches={st.kernel_launches}", flush=True)
