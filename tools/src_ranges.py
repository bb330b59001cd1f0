"""Stall breakdown per SASS address range from an ncu --page source --print-source sass CSV.

    python tools/src_ranges.py src.csv [lo-hi ...]   (offsets relative to the kernel start, hex)
Without ranges: the top instructions by samples with their stall reasons.
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
h = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith('0x')]
base = int(body[0][0], 16)
reasons = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
ci = {c: h.index(c) for c in reasons}
samp = h.index('# Samples')
exe = h.index('Instructions Executed')


def show(sel, label):
    tot = sum(int(r[samp] or 0) for r in sel)
    ins = sum(int(r[exe] or 0) for r in sel)
    st = {c: sum(int(r[ci[c]] or 0) for r in sel) for c in reasons}
    top = sorted(st.items(), key=lambda x: -x[1])[:8]
    print(f"{label}: samples {tot}, instr executed {ins}, " + " ".join(f"{k[6:]}={v}" for k, v in top if v))


if len(sys.argv) > 2:
    for rg in sys.argv[2:]:
        lo, hi_ = (int(x, 16) for x in rg.split('-'))
        show([r for r in body if lo <= int(r[0], 16) - base <= hi_], rg)
else:
    for r in sorted(body, key=lambda r: -int(r[samp] or 0))[:40]:
        st = sorted(((c[6:], int(r[ci[c]] or 0)) for c in reasons), key=lambda x: -x[1])[:3]
        print(f"{int(r[0], 16) - base:05x} {int(r[samp] or 0):5d} {r[1].strip()[:60]:60s} " + " ".join(f"{k}={v}" for k, v in st if v))
