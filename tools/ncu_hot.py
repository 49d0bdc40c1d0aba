"""Per-source-line warp-stall samples and executed instructions of one kernel in an
ncu --set full --import-source capture (all files), hottest first:

    python tools/ncu_hot.py REP.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
agg = collections.Counter()
ins = collections.Counter()
src = {}
fname = None
iS = iE = None
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        iS, iE = r.index("Warp Stall Sampling (All Samples)"), r.index("Instructions Executed")
        continue
    if not r or not r[0] or iS is None or len(r) <= iE:
        continue
    try:
        key = (fname, int(r[0]))
        agg[key] += int(r[iS] or 0)
        ins[key] += int(r[iE] or 0)
        src[key] = r[1][:90]
    except ValueError:
        pass
tot = sum(agg.values()) or 1
per_file = collections.Counter()
for k, v in agg.items():
    per_file[k[0]] += v
print("stall samples per file:", {f: f"{100 * v / tot:.1f}%" for f, v in per_file.most_common()})
for k, v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% {ins[k]:>12d}  {k[0]}:{k[1]}  {src[k]}")
