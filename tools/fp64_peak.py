"""FP64 / FP32 FMA-pipe peak (the roofline denominator MEASURED_PEAKS.json
lacks), with the SM clock sampled during the run (NVML, bench.ClockSampler).

  python tools/fp64_peak.py > profiles/fp64_peak_r02.jsonl

Builds tools/fp64_peak (nvcc, sm_100a) if needed, runs it once while sampling
clocks, and appends one summary line: best burst DFMA / FFMA, the sustained
figures, the median SM clock under load, throttle reasons, and the per-clock
rate (flop per SM per cycle: 128 = the 64 DFMA/clk/SM datasheet rate)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)


def main():
    exe = os.path.join(HERE, "fp64_peak")
    src = exe + ".cu"
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", src, "-o", exe], check=True)
    from bench import ClockSampler
    with ClockSampler(0) as clk:
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    rows = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    for r in rows:
        print(json.dumps(r))
    c = clk.summary()
    sms = rows[0]["sms"]
    best = lambda k: max((r["tflops"] for r in rows if r.get("kernel") == k), default=None)
    summ = {"summary": True, "dfma_burst_tflops": best("dfma"), "dfma_sustained_tflops": best("dfma_sustained"),
            "ffma_burst_tflops": best("ffma"), "ffma_sustained_tflops": best("ffma_sustained"), "clocks": c}
    if c.get("sm_mhz"):
        summ["dfma_flop_per_sm_per_clk_sustained"] = summ["dfma_sustained_tflops"] * 1e12 / (sms * c["sm_mhz"] * 1e6)
        summ["dfma_nominal_at_max_clock_tflops"] = sms * 128 * c["sm_max_mhz"] * 1e6 / 1e12
    print(json.dumps(summ))


if __name__ == "__main__":
    main()
