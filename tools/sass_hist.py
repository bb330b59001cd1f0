import csv, sys, collections, re
f = sys.argv[1]
rows = list(csv.reader(open(f)))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
h = rows[hi]
ie = h.index('Instructions Executed'); src = h.index('Source')
st = h.index('Warp Stall Sampling (All Samples)')
ops = collections.Counter(); stalls = collections.Counter(); tot = 0
lines = []
for r in rows[hi+1:]:
    if len(r) <= ie or r[0] == 'Address': continue
    try: n = int(r[ie])
    except: continue
    s = r[src].strip()
    op = re.sub(r'^@!?U?P\w+\s+', '', s).split(' ')[0]
    ops[op] += n; tot += n
    stalls[op] += int(r[st] or 0)
    lines.append((n, int(r[st] or 0), r[0], s))
print('total warp instr', tot)
for op, n in ops.most_common(40):
    print(f'{op:28s} {n:12d} {n/tot*100:5.1f}%  stall-samples {stalls[op]}')
if len(sys.argv) > 2:
    for n, s_, a, s in sorted(lines, key=lambda x: -x[1])[:int(sys.argv[2])]:
        print(n, s_, a[-5:], s)
