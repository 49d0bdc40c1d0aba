"""Per-CUDA-source-line executed instructions (per warp-step) and stall
samples from an ncu --set full --import-source capture:

    python tools/ncu_lines.py REP.ncu-rep WARP_STEPS [min_per_step] [lo_line hi_line]
"""
import collections
import csv
import io
import subprocess
import sys

rep, ws = sys.argv[1], float(eval(sys.argv[2]))
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
lo, hi = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (0, 10 ** 9)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi_row = next(i for i, r in enumerate(rows[:20]) if "Instructions Executed" in r)
h = rows[hi_row]
iE, iS = h.index("Instructions Executed"), 4
agg, fname = collections.OrderedDict(), None
for r in rows:
    if len(r) >= 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if len(r) <= iE or not r[0] or r[0] == "Line No":
        continue
    try:
        agg[(fname, int(r[0]), r[1][:110])] = (int(r[iE]) if r[iE] not in ("-", "") else 0,
                                                int(r[iS]) if r[iS] not in ("-", "") else 0)
    except ValueError:
        pass
st = sum(v[1] for v in agg.values()) or 1
tot = sum(v[0] for v in agg.values())
print(f"total {tot / ws:.1f} instructions per warp-step")
for k, v in sorted(agg.items(), key=lambda kv: kv[0][1]):
    if lo <= k[1] <= hi and v[0] / ws >= mn:
        print(f"{v[0] / ws:7.2f}/step {100 * v[1] / st:5.1f}% stall  {k[1]:5d}: {k[2]}")
