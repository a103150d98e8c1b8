"""Single-launch run vs the multi-launch loop on the small config-5 shapes (dev tool):
whole-step us per macro step and launches of 20-step device runs; PD_RUN_WAVES=n forces
up to n units per co-resident warp (unset: the rule in launch_fast_run)."""
import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Engine, Problem
base, _ = configs.load("c5_sweep")
tag = os.environ.get("PD_RUN_WAVES", "auto")
for nodes, lps in ((16, (12, 13)), (8, (13, 14, 15))):
    for lp in lps:
        row = []
        for K in (10, 50, 200):
            P = Problem(configs.sweep_desc(base, lp, nodes, K))
            E = Engine.from_problem(P)
            U0 = P.initial_field()
            dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
            E.run_device(dU.data_ptr(), dS.data_ptr(), 3)
            best = 1e9
            for _ in range(3):
                dU.copy_(torch.from_numpy(U0.ravel())); torch.cuda.synchronize()
                st = E.run_device(dU.data_ptr(), dS.data_ptr(), 20)
                best = min(best, st.device_ms / 20 * 1e3)
            row.append(f"K={K} {best:7.1f} us ({st.kernel_launches} launches)")
        print(f"waves={tag} {nodes}x{nodes} 2^{lp}: " + " | ".join(row), flush=True)
