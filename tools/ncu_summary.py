"""Summarise an ncu report: key metrics + per-opcode instruction mix (per state) of the top kernel.
usage: python tools/ncu_summary.py report.ncu-rep [states]"""
import csv, collections, io, subprocess, sys

rep = sys.argv[1]
states = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0 ** 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__warps_eligible.avg.per_cycle_active"]
out = {}
for k, un, x in zip(h, units, v):
    if k in want:
        out[k] = (x, un)
for k in want:
    if k in out:
        x, un = out[k]
        print(f"{k} = {x}" + (f" {un}" if un else ""))
print("-- stall reasons (per issue):")
for k, x in zip(h, v):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            if float(x) > 0.05:
                print(f"  {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:24s} {float(x):.3f}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ia, isrc = hh.index("Instructions Executed"), hh.index("Source")
tot = 0
by = collections.Counter()
for row in rows[2:]:
    try:
        nexec = int(row[ia])
    except (ValueError, IndexError):
        continue
    tot += nexec
    toks = row[isrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    by[op.split(".")[0]] += nexec
print(f"-- instruction mix: {tot:.4g} warp-instr, {tot * 32 / states:.3f} thread-instr/state")
for op, nexec in by.most_common(14):
    print(f"  {op:10s} {nexec * 32 / states:.3f}/state")
