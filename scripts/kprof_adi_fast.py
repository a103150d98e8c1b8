"""FAST ADI step launches on the 16 129-patch cdr-var case for ncu (dev tool):
python scripts/kprof_adi_fast.py [nodes-1 (10)] [nt (2)]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2405_08764_b200 import abi, configs  # noqa: E402
from paper_2405_08764_b200.engine import Engine, Problem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 2
base, _ = configs.load("ref_table1_cdr_const")
P = Problem(configs.copy_desc(base, problem=abi.PD_PROBLEM_REF_CDR_VAR, N_xi=128, N_eta=128, nx=n, ny=n, nt=nt,
                              Nt=1000, T=0.01))
E = Engine.from_problem(P, mode=abi.PD_MODE_FAST)
U0 = P.initial_field()
b, s = P.boundary_table(0.0, 4), P.source_time(0.0, 4)
U, st = E.run(U0, 4, bnd=b, src_time=s)
print("fast adi ms/step", st.device_ms / 4)
