"""Linear-response path (GapToothEngine::step with linear_cache) on the B200 vs the
unmodified reference's own fast path on one host core.  Writes profiles/<tag>_linear_path.jsonl.

  python scripts/bench_linear.py [steps] [tag]
"""
import json, sys, time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_2405_08764_b200 import configs  # noqa: E402
from paper_2405_08764_b200.engine import Engine, Problem  # noqa: E402
from oracle.pyoracle import Reference, reference_available  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
out = []
for name in ["c1_diffusion", "c3_annulus", "ref_annulus_16x10"]:
    P = Problem(configs.load(name)[0])
    E = Engine.from_problem(P)
    t0 = time.perf_counter()
    E.set_linear()
    build_s = time.perf_counter() - t0
    U0 = P.initial_field()
    E.run(U0, 10)  # warm-up
    U, st = E.run(U0, steps)
    rec = {"workload": name, "patches": E.P, "macro_steps": steps, "gpu_weights_build_s": build_s,
           "gpu_device_ms_per_macro_step": st.device_ms / steps,
           "gpu_patch_updates_per_s": E.P * steps / (st.device_ms * 1e-3), "kernel_launches_per_step": st.kernel_launches / steps}
    if reference_available():
        R = Reference().engine(P.desc, linear_cache="auto")
        Ur = R.initial_field()
        t0 = time.perf_counter()
        Ur = R.projective_step(Ur, 0.0)  # first call builds the row weights
        rec["ref_first_step_s"] = time.perf_counter() - t0
        n = min(steps, 2000)
        Ur, sec = R.steps(Ur, 1, n)
        rec["ref_ms_per_macro_step"] = 1e3 * sec / n
        rec["ref_patch_updates_per_s"] = E.P * n / sec
        rec["ref_cores"] = 1
    out.append(rec)
    print(json.dumps(rec), flush=True)
(ROOT / "profiles" / f"{sys.argv[2] if len(sys.argv) > 2 else 'r02'}_linear_path.jsonl").write_text("".join(json.dumps(r) + "\n" for r in out))
