"""Summarise an ncu report: key metrics + per-opcode instruction mix (per state) of the top kernel.
usage: python tools/ncu_summary.py report.ncu-rep [states] [--record WORKLOAD]

--record appends the kernel's figures to profiles/kernel_records.json keyed by the sha256 of the
kernel's SASS in the in-tree libqubrute_b200.so (bench.py reads instructions/state and DRAM bytes
from there only while the SASS still matches)."""
import csv, collections, io, json, os, re, subprocess, sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
args = [a for a in sys.argv[1:]]
record = None
if "--record" in args:
    i = args.index("--record")
    record = args[i + 1]
    del args[i:i + 2]
rep = args[0]
states = float(args[1]) if len(args) > 1 else 2.0 ** 40
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

if record:
    from bench import imm_sass_sha256, imm_symbol, kernel_symbol, sass_sha256

    name = out["Kernel Name"][0]
    m = re.search(r"(\w+)<([\w, ]+)>", name)
    fam, targs = m.group(1), [t.strip() for t in m.group(2).split(",")]
    lib_path = os.path.join(ROOT, "paper_2310_19373_b200", "libqubrute_b200.so")
    if fam == "coarse_kernel" and len(targs) > 6 and targs[6] in ("true", "1"):  # patched-immediate kernel (embedded cubin)
        sym, sha = imm_symbol(int(targs[4])), imm_sass_sha256(int(targs[4]))
    elif fam == "coarse2_kernel":  # super-block patched-immediate kernel (embedded cubin)
        sym, sha = imm_symbol(int(targs[2]), 2), imm_sass_sha256(int(targs[2]), 2)
    elif fam in ("coarse8_kernel", "coarse8s_kernel") and not (len(targs) > 8 and targs[8] in ("true", "1")):
        # byte-packed threshold kernels with patched immediates (embedded cubins)
        kind = (4 if fam == "coarse8s_kernel" else 3) + (2 if targs[6] in ("true", "1") else 0)
        if fam == "coarse8s_kernel" and len(targs) > 7 and targs[7] == "2":
            kind = 7
        sym, sha = imm_symbol(int(targs[4]), kind), imm_sass_sha256(int(targs[4]), kind)
    else:
        sym = kernel_symbol(lib_path, fam, int(targs[4]))
        sha = sass_sha256(lib_path, sym)
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = sum(float(out[k][0]) * scale[out[k][1]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    path = os.path.join(ROOT, "profiles", "kernel_records.json")
    recs = json.load(open(path)) if os.path.exists(path) else {}
    recs[sha] = {"kernel": sym, "kernel_name": name, "workload": record, "states": states,
                 "thread_instr_per_state": tot * 32 / states, "warp_instr": tot,
                 "issue_active_pct": float(out["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
                 "duration_ms": float(out["gpu__time_duration.sum"][0]) * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
                                                                           "second": 1e3}[out["gpu__time_duration.sum"][1]],
                 "dram_bytes_per_launch": dram, "capture": os.path.basename(rep)}
    with open(path, "w") as fh:
        json.dump(recs, fh, indent=1, sort_keys=True)
    print(f"recorded {sym} sha {sha[:16]} -> {path}")
