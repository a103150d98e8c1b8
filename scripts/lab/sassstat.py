"""Static register-read model of a SASS loop: per DP instruction, 64-bit register
operand reads (minus reuse-cache hits: same register, same slot, previous DP
instruction carried .reuse on it).  usage: sassstat.py file.sass [loop_start_hex loop_end_hex]"""
import re, sys
lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
# find the loop: the last backward BRA whose target is before it, longest body
best = None
for a, t in ins:
    m = re.search(r'BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)', t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and (best is None or a - tgt > best[1] - best[0]):
            best = (tgt, a)
lo, hi = best if len(sys.argv) < 3 else (int(sys.argv[2], 16), int(sys.argv[3], 16))
body = [(a, t) for a, t in ins if lo <= a <= hi]
from collections import Counter
op = Counter(t.split()[0].lstrip('@!P0123456789 ') if not t.startswith('@') else t.split()[1] for a, t in body)
reads = 0; hits = 0; ndp = 0; prev = {}
for a, t in body:
    toks = t.split(None, 1)
    opc = toks[0] if not toks[0].startswith('@') else t.split()[1]
    if not opc.startswith(('DFMA', 'DADD', 'DMUL')):
        continue
    ndp += 1
    args = t.split(None, 1)[1] if not toks[0].startswith('@') else t.split(None, 2)[2]
    ops = [x.strip() for x in args.split(',')]
    srcs = ops[1:]
    cur = {}
    for slot, s in enumerate(srcs):
        m = re.match(r'-?\|?(R\d+)\|?(\.reuse)?', s)
        if not m or m.group(1) == 'RZ':
            continue
        r = m.group(1)
        if prev.get(slot) == r:
            hits += 1
        else:
            reads += 1
        if m.group(2):
            cur[slot] = r
    prev = cur
print(f"loop {lo:#x}-{hi:#x}: {len(body)} instr, DP {ndp}, ops {dict(op.most_common(8))}")
shfl = sum(1 for a, t in body if 'SHFL' in t)
print(f"64-bit reg reads {reads} (+ reuse hits {hits}), SHFL32 {shfl} -> RF cycles {reads + shfl/2:.0f} vs DP pipe {2*ndp}"
      f" -> pipe util bound {min(1, 2*ndp/(reads + shfl/2)):.3f}")
