"""On-device mesh/metric generation against the host tables.

For each workload: time to a ready engine with host-sampled tables
(pd_problem_create + pd_engine_create: OpenMP sampling, H2D copy, fold) and
with coeff_gen = PD_COEFF_DEVICE (reduction pass + in-place generation + fold);
the generator kernel alone (CUDA events, ns per micro node) against what
streaming the folded table costs per node and macro step at the measured HBM
bandwidth (the in-kernel alternative SURVEY 8f #2 proposes); and the parity of
the device table with the host table.  One JSON line per workload.
usage: bench_coeffgen.py [out.jsonl]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402

from paper_2405_08764_b200 import abi, configs  # noqa: E402
from paper_2405_08764_b200.engine import Engine, Problem, generate_coeffs  # noqa: E402

_PEAKS = os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")
HBM_GBS = json.load(open(_PEAKS)).get("hbm_gbs", 6548.8) if os.path.exists(_PEAKS) else 6548.8


def ready(d):
    t0 = time.perf_counter()
    P = Problem(d)
    t1 = time.perf_counter()
    E = Engine.from_problem(P)
    t2 = time.perf_counter()
    return P, E, t1 - t0, t2 - t1


def main():
    out = open(sys.argv[1], "a") if len(sys.argv) > 1 else sys.stdout
    base4, _ = configs.load("c4_shear")
    base5, _ = configs.load("c5_sweep")
    work = [("c4_shear", base4), ("c2_cdr_tanh", configs.load("c2_cdr_tanh")[0]),
            ("c3_annulus", configs.load("c3_annulus")[0])]
    for k, nodes in ((18, 16), (20, 8), (18, 32), (20, 16)):
        work.append((f"c5_2^{k}_{nodes}x{nodes}", configs.sweep_desc(base5, k, nodes, 50)))
    for name, d in work:
        rec = {"workload": name}
        Ph, Eh, th_p, th_e = ready(configs.copy_desc(d, coeff_gen=abi.PD_COEFF_HOST))
        rec.update(patches=Eh.P, micro_nodes=f"{Eh.n1}x{Eh.n2}", host_problem_s=th_p, host_engine_s=th_e,
                   host_device_gb=Eh.device_bytes / 1e9)
        ed_h = Ph.engine_desc()
        S, n1, n2 = ed_h.ncoeff_sets, ed_h.nx + 1, ed_h.ny + 1
        small = S * n1 * n2 <= 2 ** 26
        co_h = np.ctypeslib.as_array(ed_h.coeffs, shape=(S, abi.PD_NCOEF, n1, n2)).copy() if small else None
        del Eh, Ph
        Pd, Ed, td_p, td_e = ready(configs.copy_desc(d, coeff_gen=abi.PD_COEFF_DEVICE))
        rec.update(device_problem_s=td_p, device_engine_s=td_e, device_device_gb=Ed.device_bytes / 1e9)
        rec["speedup_to_ready_engine"] = (th_p + th_e) / (td_p + td_e)
        ed = Pd.engine_desc()
        ms = []
        for _ in range(3):
            _, _, st = generate_coeffs(ed, tables=False)
            ms.append(st["device_ms"])
        nodes_ = st["nodes"]
        ns = min(ms) * 1e6 / nodes_
        n_c = 6 if st["max_abs_b"] > 0 else 5
        stream_ns = 8 * n_c / HBM_GBS  # bytes per node / (GB/s) = ns
        rec.update(generator_ms=min(ms), generator_ns_per_node=ns, stream_ns_per_node=stream_ns,
                   generator_vs_stream=ns / stream_ns, nodes=nodes_)
        if co_h is not None:
            co_d, _, _ = generate_coeffs(ed)
            rec["bit_identical_frac"] = float(np.mean(co_d == co_h))
            rec["max_rel_diff_per_coef"] = [float(np.abs(co_d[:, c] - co_h[:, c]).max() / max(np.abs(co_h[:, c]).max(), 1e-300))
                                           for c in range(abi.PD_NCOEF)]
        del Ed, Pd
        print(json.dumps(rec), file=out, flush=True)


if __name__ == "__main__":
    main()
