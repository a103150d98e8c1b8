"""Config 4 at its stated size (512x512 patches of 16x16, K = 50, 100 macro steps)
on the GPU against the committed oracle fixture: prints the relative max-norm
errors of FAST and EXACT after the first step and after the full run."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2405_08764_b200 import abi, configs  # noqa: E402
from paper_2405_08764_b200.engine import Engine, Problem  # noqa: E402

fx = np.load(ROOT / "tests" / "golden" / "c4_full.npz")
P = Problem(configs.load("c4_shear")[0])
U0 = P.initial_field()
out = {}
for name, mode in (("fast", abi.PD_MODE_FAST), ("exact", abi.PD_MODE_EXACT)):
    E = Engine.from_problem(P, mode=mode)
    U1 = E.projective_step(U0, 0.0)
    UT, st = E.run(U0, int(fx["nsteps"]))
    rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())
    out[name] = {"rel_err_step1": rel(U1, fx["U1"]), "rel_err_final": rel(UT, fx["final"]),
                 "bit_identical_final": bool(np.array_equal(UT, fx["final"])), "steps": st.steps_done,
                 "device_ms": st.device_ms}
    del E
print(json.dumps({"workload": "c4_shear full run (262144 patches, 100 macro steps)", **out}))
