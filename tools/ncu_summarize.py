"""Summarise an `ncu --set full --import-source on` capture of the fused
kernel for profiles/: the details page, DRAM traffic (JSON read by bench.py)
and the executed-instruction mix per integration step.

    python tools/ncu_summarize.py REP.ncu-rep OUT_PREFIX "workload label" STEPS_PER_LAUNCH_WARPS

STEPS_PER_LAUNCH_WARPS = warps x integration steps of the captured launch
(e.g. 3125 x 40320 for 100k patients x 4 weeks at dt 60 s); it converts
executed warp-instructions into instructions per step.
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

rep, prefix, label = sys.argv[1], sys.argv[2], sys.argv[3]
warp_steps = float(eval(sys.argv[4])) if len(sys.argv) > 4 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout


details = ncu("--page", "details", "--csv")
rows = list(csv.reader(io.StringIO(details)))
hdr = rows[0]
iname, isec, imet, iunit, ival = (hdr.index(k) for k in ("Kernel Name", "Section Name", "Metric Name",
                                                         "Metric Unit", "Metric Value"))
lines = [f"# ncu --set full: {label}", ""]
kernel = rows[1][iname] if len(rows) > 1 else "?"
lines.append(f"kernel: {kernel}")
sec = None
for r in rows[1:]:
    if r[isec] != sec:
        sec = r[isec]
        lines.append(f"\n[{sec}]")
    lines.append(f"  {r[imet]:<60s} {r[ival]} {r[iunit]}")

raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
get = lambda name: float(v[h.index(name)].replace(",", "")) if name in h else None
traffic = {"kernel": kernel, "workload": label,
           "dram_bytes_read": get("dram__bytes_read.sum"), "dram_bytes_write": get("dram__bytes_write.sum"),
           "duration_ns": get("gpu__time_duration.sum"), "source": f"ncu --set full ({prefix}_ncu.txt)"}
# ncu reports MB / GB in raw units for some versions; normalise to bytes
unit_row = raw[1]
for k, name in (("dram_bytes_read", "dram__bytes_read.sum"), ("dram_bytes_write", "dram__bytes_write.sum")):
    u = unit_row[h.index(name)] if name in h else ""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    if traffic[k] is not None:
        traffic[k] = int(traffic[k] * scale)
if traffic["duration_ns"] is not None:
    u = unit_row[h.index("gpu__time_duration.sum")]
    traffic["duration_ns"] *= {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "s": 1e9}.get(u, 1)
json.dump(traffic, open(f"{prefix}_traffic.json", "w"), indent=1)

# pipe utilisation: the counters north_star asks for (FP64 / FP32 pipes, plus
# the SFU = XU pipe) and the issue rate that bounds an issue-limited kernel
PIPES = [
    ("fp64_pipe_cycles_active_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("fp64_inst_executed_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    ("fma_pipe_cycles_active_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("fmaheavy_pipe_cycles_active_pct", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("fma_inst_executed_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    ("alu_pipe_cycles_active_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    ("xu_sfu_inst_executed_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("lsu_inst_executed_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("ipc_per_sm", "sm__inst_executed.avg.per_cycle_active"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("dram_throughput_pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
]


def _num(name):
    try:
        return get(name)
    except ValueError:
        return None


pipes = {"kernel": kernel, "workload": label, "source": f"ncu --set full ({prefix}_ncu.txt)"}
for key, name in PIPES:
    pipes[key] = _num(name)
json.dump(pipes, open(f"{prefix}_pipes.json", "w"), indent=1)
lines.insert(3, "\n[pipe utilisation]")
for i, (key, name) in enumerate(PIPES):
    val = pipes[key]
    lines.insert(4 + i, f"  {key:<34s} {'n/a' if val is None else f'{val:.2f}'}   ({name})")

src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
sh = src[1]
iS, iE = sh.index("Source"), sh.index("Instructions Executed")
ops, tot = collections.Counter(), 0
for r in src[2:]:
    try:
        e = int(r[iE])
    except (ValueError, IndexError):
        continue
    s = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip())
    op = s.split()[0].split(".")[0] if s else "?"
    ops[op] += e
    tot += e
lines.append("\n[executed instruction mix]")
lines.append(f"  total warp-instructions {tot}" + (f"  = {tot / warp_steps:.1f} per warp-step" if warp_steps else ""))
for op, c in ops.most_common(30):
    per = f"{c / warp_steps:7.2f}/step" if warp_steps else ""
    lines.append(f"  {op:<10s} {100 * c / tot:6.2f} %  {per}")
# warp-state sampling: where the warps wait (latency vs issue)
stalls = []
for k, x in zip(h, v):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
        try:
            stalls.append((float(x.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot_s = sum(c for c, _ in stalls) or 1.0
lines.append("\n[warp-state samples (smsp__pcsamp_warps_issue_stalled_*)]")
for c, k in sorted(stalls, reverse=True):
    if c > 0:
        lines.append(f"  {k:<28s} {100 * c / tot_s:5.1f} %")
open(f"{prefix}_ncu.txt", "w").write("\n".join(lines) + "\n")
print(f"wrote {prefix}_ncu.txt, {prefix}_traffic.json, {prefix}_pipes.json; {tot / warp_steps if warp_steps else tot:.1f}")
