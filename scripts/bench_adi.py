"""ADI micro-solver on the B200 (EXACT and FAST families) vs the unmodified reference on one host core.
Writes profiles/r01_adi.jsonl (or the path given).   python scripts/bench_adi.py [out.jsonl]"""
import json, sys, time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2405_08764_b200 import abi, configs  # noqa: E402
from paper_2405_08764_b200.engine import Engine, Problem  # noqa: E402
from oracle.pyoracle import Reference, reference_available  # noqa: E402

base, _ = configs.load("ref_table1_cdr_const")
cases = [
    ("table1 cdr-const N=10 (81 patches 11x11, nt=2, upwind two)", {}, 1001),
    ("table3 cdr-var lambda=0.3 N=10, Nt=2000 (upwind four)",
     {"problem": abi.PD_PROBLEM_REF_CDR_VAR, "lambda_": 0.3, "upwind_order": abi.PD_UPWIND_FOUR, "Nt": 2000}, 2000),
    ("cdr-var N=128 (16129 patches 11x11, nt=2)", {"problem": abi.PD_PROBLEM_REF_CDR_VAR, "N_xi": 128, "N_eta": 128,
                                                     "Nt": 1000, "T": 0.01}, 50),
    ("cdr-var N=128, 21x21 nodes, nt=4", {"problem": abi.PD_PROBLEM_REF_CDR_VAR, "N_xi": 128, "N_eta": 128,
                                          "nx": 20, "ny": 20, "nt": 4, "Nt": 1000, "T": 0.01}, 40),
]
out = []
for label, over, steps in cases:
    P = Problem(configs.copy_desc(base, **over))
    U0 = P.initial_field()
    bnd, src = P.boundary_table(0.0, steps), P.source_time(0.0, steps)
    n1, n2, nt = P.desc.nx + 1, P.desc.ny + 1, P.desc.nt
    rec = {"workload": label, "micro_nodes": n1 * n2, "nt": nt, "macro_steps": steps}
    for fam, mode in (("exact", abi.PD_MODE_EXACT), ("fast", abi.PD_MODE_FAST)):
        E = Engine.from_problem(P, mode=mode)
        E.run(U0, 3, bnd=bnd[:3], src_time=src[:3])
        U, st = E.run(U0, steps, bnd=bnd, src_time=src, raise_on_instability=False)
        assert st.steps_done == steps, f"{label} {fam}: macro guard tripped at step {st.failed_step}"
        upd = E.P * n1 * n2 * nt
        rec["patches"] = E.P
        rec[f"gpu_{fam}_ms_per_macro_step"] = st.device_ms / steps
        rec[f"gpu_{fam}_node_updates_per_s"] = upd * steps / (st.device_ms * 1e-3)
        rec[f"gpu_{fam}_kernel_family"] = "exact" if E.mode == abi.PD_MODE_EXACT else "fast"
    if reference_available():
        R = Reference().engine(P.desc)
        Ur = R.initial_field()
        n = max(2, min(steps, int(2.0 / max(1e-9, 1.6e-3 * E.P / 81))))  # ~2 s of reference time
        Ur, sec = R.steps(Ur, 0, n)
        rec.update({"ref_ms_per_macro_step": 1e3 * sec / n, "ref_node_updates_per_s": upd * n / sec,
                    "ref_cores": 1, "ref_sample_steps": n})
    out.append(rec)
    print(json.dumps(rec), flush=True)
(Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r01_adi.jsonl").write_text("".join(json.dumps(r) + "\n" for r in out))
