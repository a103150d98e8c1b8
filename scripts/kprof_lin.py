import sys
sys.path.insert(0, "/root/repo")
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Engine, Problem
name = sys.argv[1] if len(sys.argv) > 1 else "c1_diffusion"
P = Problem(configs.load(name)[0])
E = Engine.from_problem(P)
E.set_linear()
U0 = P.initial_field()
for _ in range(2):
    U, st = E.run(U0, 2000)
print(name, "us/step", 1e3 * st.device_ms / 2000)
