import re, sys
lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', ln)
    if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
body = [(a, t) for a, t in ins if lo <= a <= hi]
def parse(t):
    p = t.split(None, 1)
    if not p[0].startswith(('DFMA', 'DADD', 'DMUL')): return None
    ops = [x.strip() for x in p[1].split(',')]
    srcs = [re.sub(r'[-|]|\.reuse', '', s) for s in ops[1:]]
    return p[0], ops[0], srcs
prev = None; same = 0; swap = 0; any_adj = 0; skip_nondp = 0
for a, t in body:
    q = parse(t)
    if q is None:
        continue
    if prev is not None:
        op, d, s = q; pop, pd, ps = prev
        shared = set(x for x in s if x.startswith('R') and x != 'RZ') & set(x for x in ps if x.startswith('R') and x != 'RZ')
        if shared:
            any_adj += 1
            r = shared.pop()
            if s.index(r) == ps.index(r): same += 1
            elif op == 'DFMA' and pop == 'DFMA' and {s.index(r), ps.index(r)} == {0, 1}: swap += 1
    prev = q
print(f"adjacent DP pairs sharing a source: {any_adj}; same slot: {same}; fixable by A<->B swap: {swap}")
