"""Summarise an ncu --set full report of the fused step kernel into profiles/ (dev tool).

usage: ncu_summarize.py REPORT.ncu-rep KEY KERNEL_DESC ALG_BYTES SOURCE_TXT
Writes/updates profiles/ncu_summary.json[KEY] (bench.py reads dram_bytes_per_launch from it) and
dumps the details page to profiles/SOURCE_TXT."""
import csv, io, json, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep, key, desc, alg, txt = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
m = {}
for k in want:
    if k in hdr:
        i = hdr.index(k)
        m[k] = {"value": float(vals[i].replace(",", "")), "unit": units[i]}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = m["dram__bytes_read.sum"]["value"] * scale[m["dram__bytes_read.sum"]["unit"]]
wr = m["dram__bytes_write.sum"]["value"] * scale[m["dram__bytes_write.sum"]["unit"]]
p = ROOT / "profiles" / "ncu_summary.json"
d = json.loads(p.read_text()) if p.exists() else {}
d[key] = {"kernel": desc, "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
          "algorithmic_bytes_per_launch": alg,
          "source": f"profiles/{txt} (ncu --set full --clock-control none, one launch)", "metrics": m}
p.write_text(json.dumps(d, indent=1) + "\n")
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True, check=True).stdout
(ROOT / "profiles" / txt).write_text(det)
print(key, "dram/launch", rd + wr, "alg", alg)
