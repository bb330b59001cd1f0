"""List the loops (backward branches) of one kernel in a cuobjdump -sass dump.

    cuobjdump -sass lib.so > all.sass; python tools/sass_loops.py all.sass ws_kernelILi1Eh
Prints each loop's body size and opcode histogram (innermost first).
"""
import collections
import re
import sys

text = open(sys.argv[1]).read().split("Function : ")
fn = [t for t in text if t.split("\n", 1)[0].find(sys.argv[2]) >= 0][0]
ins = []
for line in fn.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
    if m and m.group(1):
        tgt = int(m.group(1), 16)
        if tgt <= a and tgt in addr:
            loops.append((addr[tgt], i))
print(f"{len(ins)} instructions, {len(loops)} backward branches")
for s, e in sorted(loops, key=lambda x: x[1] - x[0]):
    body = [t for _, t in ins[s:e + 1]]
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in body)
    print(f"loop {ins[s][0]:05x}-{ins[e][0]:05x}: {len(body)} instr  " +
          " ".join(f"{k}:{v}" for k, v in ops.most_common(14)))
