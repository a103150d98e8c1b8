"""Device us per macro step of the single-launch run (k_fast_run) on configs 1-3
and the small config-5 points, best of three 200-step runs (dev tool for A/B
of library builds: scripts/ab.sh run tagA tagB)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_08764_b200 import configs  # noqa: E402
from paper_2405_08764_b200.engine import Engine, Problem  # noqa: E402

cases = [(n, configs.load(n)[0]) for n in ("c1_diffusion", "c2_cdr_tanh", "c3_annulus")]
base, _ = configs.load("c5_sweep")
for lp, nodes, K in [(12, 8, 10), (12, 16, 10), (13, 8, 10), (12, 8, 50), (14, 8, 10)]:
    cases.append((f"c5-2^{lp}-{nodes}-K{K}", configs.sweep_desc(base, lp, nodes, K)))
out = []
for name, d in cases:
    P = Problem(d)
    E = Engine.from_problem(P)
    n = 200
    U0 = P.initial_field()
    b = P.boundary_table(0.0, n)
    best = min(E.run(U0, n, bnd=b)[1].device_ms / n for _ in range(3))
    out.append(f"{name} {1e3 * best:.2f}")
print("run us/step: " + " | ".join(out), flush=True)
