"""Summarise an ncu SASS source-page CSV: executed instructions by opcode
class and the hottest instructions with their stall reasons."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
ops = collections.Counter()
stalls = collections.Counter()
tot = 0
for r in data:
    try:
        n = int(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        continue
    src = r[idx["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    ops[op.split(".")[0]] += n
    tot += n
    for k, i in idx.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                stalls[k] += int(r[i] or 0)
            except ValueError:
                pass
print("total executed warp-instructions", tot)
for op, n in ops.most_common(40):
    print(f"{op:12s} {n:14d} {100 * n / tot:6.2f}%")
print("stalls (samples):")
st = sum(stalls.values())
for k, v in stalls.most_common(12):
    print(f"  {k:28s} {v:10d} {100 * v / max(st, 1):6.2f}%")
