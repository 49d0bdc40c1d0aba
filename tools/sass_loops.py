"""List the innermost backward-branch loops of one kernel in a cuobjdump
-sass dump, with the opcode histogram of each loop body.

    python tools/sass_loops.py dump.sass <function-substring> [min_len] [max_len]
"""
import collections
import re
import sys

text = open(sys.argv[1]).read()
key = sys.argv[2]
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 100
hi = int(sys.argv[4]) if len(sys.argv) > 4 else 400
funcs = re.split(r"\n\s*Function : ", text)
body = next(f for f in funcs[1:] if key in f.split("\n", 1)[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, s) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*)?(0x[0-9a-f]+)", s)
    if not m:
        continue
    t = int(m.group(1), 16)
    if t < a and t in addr_idx:
        j = addr_idx[t]
        n = i - j + 1
        if lo <= n <= hi:
            ops = collections.Counter()
            for _, x in ins[j:i + 1]:
                x = re.sub(r"^@!?U?P[T0-9]+\s+", "", x)
                ops[x.split()[0].split(".")[0]] += 1
            print(f"loop {t:#x}..{a:#x}: {n} instructions")
            print("   ", ", ".join(f"{k} {v}" for k, v in ops.most_common()))
