"""ALU / issue-slot peaks for the roofline denominators, with the SM clock sampled while they run.

Runs tools/alu_peaks (built here if missing) once per kernel, each for ~1 s of back-to-back
launches, while nvidia-smi samples the SM clock and throttle reasons (bench.ClockSampler).  The
per-SM-per-clock figures divide the CUDA-event rate by the SMs and the MEDIAN SAMPLED clock, so
they are bounded by the architecture (128 FP32 lanes, 4 warp-instructions issued per SM per clock)
when the measurement is sound -- the check the r01 capture (clock64-derived) failed.

    python tools/alu_peaks.py [--out profiles/r12_alu_peaks.json]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

from bench import ClockSampler  # noqa: E402

BIN = os.path.join(ROOT, "tools", "alu_peaks")
SRC = BIN + ".cu"
NAMES = ["fadd", "fadd2", "ffma", "fmnmx3", "dadd", "iadd3", "vimnmx3", "mix_fadd2_fmnmx3_ldcu128", "viadd_16x2",
         "vimnmx3_s16x2", "mix16_viadd2_vimnmx3_ldcu128", "issue_fadd_iadd3"]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r12_alu_peaks.json"))
    ap.add_argument("--seconds", type=float, default=1.5)
    args = ap.parse_args()
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", BIN, SRC])
    results = {}
    for k, name in enumerate(NAMES):
        probe = json.loads(subprocess.check_output([BIN, str(k), "20"], text=True))
        launches = max(50, int(args.seconds * 1e3 / probe["ms_per_launch"]))
        sampler = ClockSampler(0)
        sampler.start()
        time.sleep(0.3)
        rec = json.loads(subprocess.check_output([BIN, str(k), str(launches)], text=True))
        clocks = sampler.stop()
        mhz = clocks["sm_mhz"]
        sms = rec["sms"]
        if mhz:
            rec["sm_mhz_sampled"] = mhz
            rec["lane_ops_per_sm_clk"] = rec["lane_ops_per_s"] / (sms * mhz * 1e6)
            rec["warp_instr_per_sm_clk"] = rec["warp_instr_per_s"] / (sms * mhz * 1e6)
        rec["clocks"] = clocks
        results[name] = rec
        print(name, json.dumps(rec), flush=True)
    out = {
        "gpu": subprocess.run(["nvidia-smi", "--query-gpu=name", "--format=csv,noheader"], capture_output=True,
                              text=True).stdout.strip(),
        "method": "tools/alu_peaks.cu, one kernel per process, 2 CTAs x 512 threads per SM, 16 independent chains "
                  "per thread, back-to-back launches for ~%.1f s (CUDA events); SM clock = median of nvidia-smi "
                  "samples during the run (tools/alu_peaks.py)" % args.seconds,
        "results": results,
    }
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
