"""One whole-run launch (k_fast_run) of a small config for ncu: python scripts/kprof_run.py [config] [steps]"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Engine, Problem
name = sys.argv[1] if len(sys.argv) > 1 else "c1_diffusion"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
P = Problem(configs.load(name)[0])
E = Engine.from_problem(P)
U0 = P.initial_field()
b = P.boundary_table(0.0, n)
for _ in range(2):
    U, st = E.run(U0, n, bnd=b)
print(name, "ms/step", st.device_ms / n, "launches", st.kernel_launches)
