import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2405_08764_b200 import abi, configs
from paper_2405_08764_b200.engine import Engine, Problem
from oracle.pyoracle import Restated
O = Restated()
d = configs.default_desc(); d.problem = abi.PD_PROBLEM_REF_CDR
d.N_xi = d.N_eta = 10; d.Nt, d.T, d.tau = 1001, 1.0, 1e-6; d.nx = d.ny = 10; d.nt = 250
P = Problem(d); E = Engine.from_problem(P); print('mode', E.mode)
U0 = P.initial_field(); bt, stt = P.boundary_table(0.0, 4), P.source_time(0.0, 4)
st, Uo, so = O.run(P.engine_desc(), U0, 4, bnd=bt, src_time=stt); print('oracle run status', st, so.failed_step)
_, O1 = O.projective_step(P.engine_desc(), U0, 0.0, bnd=bt[0], src_time=stt[0])
G1 = E.projective_step(U0, 0.0, bnd=bt[0], src_time=stt[0])
print('single step maxdiff', np.abs(G1 - O1).max(), np.abs(O1).max(), np.abs(G1).max())
S1 = E.step_direct(U0, 0.0, src_time=stt[0, 0]); _, So = O.gaptooth_step(P.engine_desc(), U0, 0.0, src_time=stt[0,0])
print('substep maxdiff', np.abs(S1 - So).max())
Ug, sg = E.run(U0, 4, bnd=bt, src_time=stt, raise_on_instability=False)
print('run', sg.failed_step, sg.blowup_threshold, np.abs(Ug - Uo).max())
