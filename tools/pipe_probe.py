"""Run tools/pipe_probe kernels with the SM clock sampled (see pipe_probe.cu for what each pairs)."""
import json, os, subprocess, sys, time
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402
BIN = os.path.join(ROOT, "tools", "pipe_probe")
NAMES = ["imad+imad", "imad+vimnmx3", "imad+hadd2", "vimnmx3+hadd2", "imad+hmnmx2", "vimnmx3+hmnmx2",
         "hadd2+hadd2", "hmnmx2+hmnmx2", "fadd+imad", "fadd+hadd2", "coarse_mix_2imad_1vimnmx3_1viaddmnmx",
         "coarse_mix_2imad_1vimnmx3_2viaddmnmx"]
if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(BIN + ".cu"):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", BIN, BIN + ".cu"])
out = {}
for k, name in enumerate(NAMES):
    probe = json.loads(subprocess.check_output([BIN, str(k), "5"], text=True))
    launches = max(20, int(1000 / probe["ms_per_launch"]))
    s = ClockSampler(0); s.start(); time.sleep(0.3)
    rec = json.loads(subprocess.check_output([BIN, str(k), str(launches)], text=True))
    clk = s.stop()
    rec["sm_mhz"] = clk["sm_mhz"]
    rec["warp_instr_per_sm_clk"] = rec["warp_instr_per_s"] / (rec["sms"] * clk["sm_mhz"] * 1e6)
    out[name] = rec
    print(f"{name:18s} {rec['warp_instr_per_sm_clk']:.3f} warp-instr/SM/clk at {clk['sm_mhz']} MHz", flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "pipe_probe.json"), "w"), indent=1)
