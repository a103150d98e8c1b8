"""One ADI step launch (Table-1 setup) for ncu: python scripts/kprof_adi.py [N]"""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Engine, Problem
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
base, _ = configs.load("ref_table1_cdr_const")
P = Problem(configs.copy_desc(base, N_xi=N, N_eta=N))
E = Engine.from_problem(P)
U0 = P.initial_field()
b, s = P.boundary_table(0.0, 6), P.source_time(0.0, 6)
U, st = E.run(U0, 6, bnd=b, src_time=s)
print("ms/step", st.device_ms / 6)
