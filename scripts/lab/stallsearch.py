"""Lab: compile the FAST 16x16 mixed kernel (k_fast<FC16M>) under source
variants (-D macros) and report the micro-step loop's SASS statistics: the
sum of the control-word stall counts (ptxas's own cycle budget per warp and
iteration: measured kernel time per micro-step tracks it, profiles/r02_ceiling.md),
64-bit register reads and reuse hits.  Compile-only, no GPU.

usage: stallsearch.py "-DA=1 -DB=2" ["..." ...]
"""
import os, re, subprocess, sys, tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CSRC = os.path.join(ROOT, "paper_2405_08764_b200", "csrc")
KERNELS = {
    "fast16": ("_ZN6pdb2003dev6k_fastINS0_7FastCfgILi16ELi16ELi2ELi4ELb1ELb0ELb0ELb0EEEEEvNS0_6ParamsEPKdPdiPKiS6_iS9_S6_",
               '#include "kernels_fast.cuh"\nnamespace pdb200::dev {\ntemplate __global__ void k_fast<FC16M>(Params, const double*, '
               'double*, int, const int*, const double*, int, const int*, const double*);\n}\n'),
    "big32": ("_ZN6pdb2003dev10k_fast_bigINS0_6BigCfgILi32ELb1ELb0ELb0EEEEEvNS0_6ParamsEPKdPdiPKiS6_S9_",
              '#include "kernels_fast_big.cuh"\nnamespace pdb200::dev {\ntemplate __global__ void k_fast_big<BC32M>(Params, const double*, '
              'double*, int, const int*, const double*, const int*);\n}\n'),
    "fast8": ("_ZN6pdb2003dev6k_fastINS0_7FastCfgILi8ELi8ELi2ELi4ELb1ELb0ELb0ELb0EEEEEvNS0_6ParamsEPKdPdiPKiS6_iS9_S6_",
              '#include "kernels_fast.cuh"\nnamespace pdb200::dev {\ntemplate __global__ void k_fast<FC8M>(Params, const double*, '
              'double*, int, const int*, const double*, int, const int*, const double*);\n}\n'),
    "run9": ("_ZN6pdb2003dev10k_fast_runINS0_7FastCfgILi9ELi9ELi3ELi3ELb0ELb0ELb0ELb0EEEEEvNS0_6ParamsEPdS5_PKiPKdiS9_mS9_midPySA_PiS9_SA_",
             '#include "kernels_fast.cuh"\nnamespace pdb200::dev {\ntemplate __global__ void k_fast_run<FC9>(Params, double*, double*, '
             'const int*, const double*, int, const double*, size_t, const double*, size_t, int, double, unsigned long long*, '
             'unsigned long long*, int*, const double*, unsigned long long*);\n}\n'),
    "run7": ("_ZN6pdb2003dev10k_fast_runINS0_7FastCfgILi7ELi7ELi1ELi7ELb0ELb0ELb0ELb0EEEEEvNS0_6ParamsEPdS5_PKiPKdiS9_mS9_midPySA_PiS9_SA_",
             '#include "kernels_fast.cuh"\nnamespace pdb200::dev {\ntemplate __global__ void k_fast_run<FC7>(Params, double*, double*, '
             'const int*, const double*, int, const double*, size_t, const double*, size_t, int, double, unsigned long long*, '
             'unsigned long long*, int*, const double*, unsigned long long*);\n}\n'),
}
KERNEL = os.environ.get("LAB_KERNEL", "fast16")
ENTRY, TU = KERNELS[KERNEL]


def loop_stats(sass: str):
    lines = sass.splitlines()
    ins = []
    for i, l in enumerate(lines):
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/', l)
        if m:
            hi = int(re.search(r'/\* (0x[0-9a-f]+) \*/', lines[i + 1]).group(1), 16)
            ins.append((int(m.group(1), 16), m.group(2).strip(), hi))
    loops = []
    for a, t, _ in ins:
        m = re.search(r'BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)', t)
        if m:
            tg = int(m.group(1), 16)
            if tg < a:
                loops.append((tg, a))
    # the micro-step loop: the shortest backward branch whose body holds >= 20 DFMA
    def ndfma(lo, hi):
        return sum(1 for a, t, _ in ins if lo <= a <= hi and 'DFMA' in t)
    cand = [l for l in loops if ndfma(*l) >= 20]
    best = min(cand, key=lambda l: l[1] - l[0])
    body = [x for x in ins if best[0] <= x[0] <= best[1]]
    stall = sum((h >> 41) & 0xF for _, _, h in body)
    reads = hits = 0
    prev = {}
    for _, t, _ in body:
        opc = t.split()[0] if not t.startswith('@') else t.split()[1]
        if not opc.startswith(('DFMA', 'DADD', 'DMUL')):
            continue
        args = t.split(None, 1)[1] if not t.startswith('@') else t.split(None, 2)[2]
        cur = {}
        for slot, s in enumerate(x.strip() for x in args.split(',')[1:]):
            m = re.match(r'-?\|?(R\d+)\|?(\.reuse)?', s)
            if not m or m.group(1) == 'RZ':
                continue
            if prev.get(slot) == m.group(1):
                hits += 1
            else:
                reads += 1
            if m.group(2):
                cur[slot] = m.group(1)
        prev = cur
    return len(body), stall, reads, hits


def compile_variant(defs: str, regs=None):
    with tempfile.TemporaryDirectory() as d:
        cu = os.path.join(d, "one.cu")
        open(cu, "w").write(TU)
        ptx = os.path.join(d, "one.ptx")
        cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
               f"-I{ROOT}/include", f"-I{CSRC}", "-ptx", "-o", ptx, cu] + defs.split()
        subprocess.run(cmd, check=True, capture_output=True)
        cub = os.path.join(d, "one.cubin")
        pcmd = ["ptxas", "-arch=sm_100a", "-O3", f"--entry={ENTRY}", "-o", cub, ptx, "-v"]
        if regs:
            pcmd.append(f"--maxrregcount={regs}")
        r = subprocess.run(pcmd, check=True, capture_output=True, text=True)
        used = re.search(r"Used (\d+) registers", r.stderr)
        spill = re.search(r"(\d+) bytes spill stores", r.stderr)
        sass = subprocess.run(["cuobjdump", "-sass", cub], check=True, capture_output=True, text=True).stdout
        return loop_stats(sass), int(used.group(1)), int(spill.group(1)) if spill else 0


if __name__ == "__main__":
    for defs in sys.argv[1:] or [""]:
        (n, stall, reads, hits), regs, spill = compile_variant(defs)
        print(f"{defs or '(default)':60s} loop {n} instr  stall {stall}  reads {reads} hits {hits}  regs {regs} spill {spill}",
              flush=True)
