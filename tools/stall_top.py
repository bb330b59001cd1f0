"""Top instructions per stall reason from an ncu --page source --print-source sass CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
h = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != 'Address']
reasons = sys.argv[2].split(',') if len(sys.argv) > 2 else ['stall_long_sb', 'stall_wait', 'stall_short_sb', 'stall_barrier']
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
for reason in reasons:
    c = h.index(reason)
    tot = sum(int(r[c] or 0) for r in body)
    print(f'== {reason}: {tot} samples')
    for r in sorted(body, key=lambda r: -int(r[c] or 0))[:n]:
        print(f'   {int(r[c]):6d} {r[0][-5:]} {r[1].strip()[:70]}')
