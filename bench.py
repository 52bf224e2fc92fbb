"""Benchmark: QUBO states evaluated per second (2^n / solve time) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config E] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Workload (BASELINE.json configs[4]): one exhaustive solve of a
seeded n=40 instance — upper-triangular fp32 Q, 10% off-diagonal density, N(0,1)
nonzeros, dense N(0,1) diagonal — over all 2^40 states.  A "step" is one full solve;
with N ranks the chunk space is split into N equal shards (strong scaling: the total
work is fixed) and the argmin is combined with one NCCL all-reduce.

value  = 2^n * K / (max over ranks of the summed device time of the solve kernels,
         CUDA events on the library's stream); Q already packed, no host copies timed.
e2e    = the same metric through the public API (solve_incremental at N=1,
         distributed.solve_sharded at N>1) with Q in host memory: planning, the kernel
         parameter upload (H2D), the result read-back (D2H) and the collective inside the
         timed region; wall clock, max over ranks.
Timing hygiene: W warm-up steps; a 256 MiB L2 flush between timed steps; nvidia-smi clocks
sampled during the timed region.  cpu_baseline: the unmodified reference (baseline/_ref, numba,
all host threads) when staged, else its oracle port (oracle/, C), on a bounded sample of the
same workload, rank 0 at N=1; the port's figure is kept beside it (cpu_baseline_port).
--impl reference: the unmodified reference package (baseline/_ref, numba kernels) on all host
cores when it is staged, else the oracle port; each step a bounded sample (run_reference).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_DESC = {
    "A": "A: n=20 int32 U[-100,100], single instance",
    "B": "B: n=24 fp32 N(0,1), single instance",
    "D": "D: n=32 int32 U[-1000,1000], single instance",
    "E": "E: n=40 fp32 N(0,1), 10% off-diagonal density, dense diagonal",
}
# Roofline inputs.  The path is ALU-issue bound (0 algorithmic HBM bytes per state):
# * the issue-slot peak in warp-instructions per SM per clock is MEASURED by tools/alu_peaks.py
#   (FFMA + IADD3 on independent pipes, nvidia-smi-sampled clock); fallback 4 (one per SMSP per clock);
# * the instructions the dominant kernel issues per state come from an ncu capture of that kernel
#   (tools/ncu_summary.py --record), keyed by the sha256 of its SASS in the library that ran: if the
#   kernel changed since the capture, the issue figures are withheld rather than reported stale.
ALU_PEAKS = os.path.join(ROOT, "profiles", "r12_alu_peaks.json")
ISSUE_WARP_INSTR_PER_SM_CLK = 4.0
FP32_ADD_LANES_PER_SM_CLK = 128.0
KERNEL_RECORDS = os.path.join(ROOT, "profiles", "kernel_records.json")


def kernel_symbol(lib_path: str, family: str, L: int):
    """Mangled name of ``qb::<family><..., L, ...>`` in the library (5th template argument = L)."""
    import re

    try:
        out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True,
                             timeout=60).stdout
    except (OSError, subprocess.SubprocessError):
        return None
    pat = re.compile(r"_ZN2qb%d%sI(?:Li\d+E){4}Li%dE(?:L[ib]\d+E)*EEvNS_\w+E$" % (len(family), family, L))
    for line in out.split("\n"):
        parts = line.split()
        if parts and pat.match(parts[-1]):
            return parts[-1]
    return None


def sass_sha256(lib_path: str, symbol: str):
    """sha256 of the SASS instruction text of one kernel in the library (cuobjdump), or None."""
    import hashlib

    try:
        out = subprocess.run(["cuobjdump", "-sass", "-fun", symbol, lib_path], capture_output=True, text=True,
                             timeout=120).stdout
    except (OSError, subprocess.SubprocessError):
        return None
    body = [ln.strip() for ln in out.split("\n") if ln.strip().startswith("/*") and "*/" in ln]
    if not body:
        return None
    return hashlib.sha256("\n".join(body).encode()).hexdigest()


def imm_sass_sha256(L: int, kind: int = 1):
    """sha256 of the SASS of a patched-immediate coarse kernel (kind 1: 10-bit, 2: super-block, 3: byte-packed
    threshold pass, 4: its super-block form) for chunk length L with its placeholders in place (the code, independent of any instance's table
    words), or None."""
    import tempfile

    import numpy as np

    from paper_2310_19373_b200 import _lib

    try:
        img = _lib.imm_image(L, np.uint32(0x7A5C0000) | np.arange(_lib.IMM_WORDS[kind], dtype=np.uint32), kind)
    except Exception:  # noqa: BLE001 - no cubin for this L / library without the IMM kernels
        return None
    with tempfile.NamedTemporaryFile(suffix=".cubin") as fh:
        fh.write(img)
        fh.flush()
        return sass_sha256(fh.name, imm_symbol(L, kind))


def imm_symbol(L: int, kind: int = 1) -> str:
    if kind >= 3:  # byte-packed threshold kernels: 3 + super-block + 2 * row-bound form; 7: row-bound, 12-bit blocks
        nx = {4: 1, 6: 1, 7: 2}.get(kind, 0)
        fam, tail = ("15coarse8s_kernel", f"Li{nx}ELb0E") if nx else ("14coarse8_kernel", "")
        return f"_ZN2qb{fam}ILi5ELi5ELi4ELi6ELi{L}ELi128ELb{int(kind >= 5)}E{tail}EEvNS_11TableParamsE"
    if kind == 2:
        return f"_ZN2qb14coarse2_kernelILi5ELi5ELi{L}ELi128EEEvNS_11TableParamsE"
    return f"_ZN2qb13coarse_kernelILi5ELi5ELi4ELi6ELi{L}ELi128ELb1EEEvNS_11TableParamsE"


def kernel_record(sha):
    """The committed ncu record (instr/state, DRAM bytes, issue activity) for this SASS, or None."""
    try:
        with open(KERNEL_RECORDS) as fh:
            recs = json.load(fh)
    except (OSError, ValueError):
        return None
    return recs.get(sha) if sha else None


def issue_peak_per_sm_clk():
    """(warp-instructions issued per SM per clock, source): the highest rate any of the
    tools/alu_peaks.py kernels sustained on this pool's B200 (per-clock with the sampled SM clock),
    else the architectural 4 (one per SMSP per clock)."""
    try:
        with open(ALU_PEAKS) as fh:
            res = json.load(fh)["results"]
        name, rec = max(res.items(), key=lambda kv: kv[1]["warp_instr_per_sm_clk"])
        return float(rec["warp_instr_per_sm_clk"]), (f"measured ({os.path.relpath(ALU_PEAKS, ROOT)}: best issue rate, "
                                                     f"'{name}' at {rec['sm_mhz_sampled']:.0f} MHz sampled)")
    except (OSError, KeyError, ValueError, TypeError):
        return ISSUE_WARP_INSTR_PER_SM_CLK, "fallback: 4 warp-instr/SM/clk (1 per SMSP per clock)"


def fp32_lane_peak_per_sm_clk():
    try:
        with open(ALU_PEAKS) as fh:
            rec = json.load(fh)["results"]["fadd2"]
        return float(rec["lane_ops_per_sm_clk"]), "measured FADD2 lane rate"
    except (OSError, KeyError, ValueError, TypeError):
        return FP32_ADD_LANES_PER_SM_CLK, "fallback 128 FP32 lanes/SM/clk"


FAMILIES = {1: "table_kernel", 2: "fieldwalk_kernel", 3: "coarse_kernel", 4: "tc_kernel", 5: "coarse_kernel (imm)",
            6: "coarse2_kernel (imm)", 7: "coarse8_kernel (imm)", 8: "coarse8s_kernel (imm)",
            9: "coarse8_kernel (imm, row-bound)", 10: "coarse8s_kernel (imm, row-bound)",
            11: "coarse8s_kernel (imm, row-bound, 12-bit)", 12: "coarse8s_kernel"}


def roofline_block(r, n, per_launch_states, search_s, sm_count, sm_hz, lib_path):
    """Issue-slot roofline of the search kernel (the path is ALU-issue bound).

    achieved = per-launch states x (instructions per state, from the ncu record of THIS kernel's
    SASS) / 32 / the launch's CUDA-event time; peak = measured issue rate per SM per clock x SMs x
    the SM clock sampled during the timed region.  ``nominal_frac`` keeps SURVEY.md §8d's n+1
    ops/state basis against the measured FP32 lane rate: > 1 because the table method forms a
    state's value with ~1 instruction instead of n+1 additions."""
    L = n - int(r.prefix_bits)
    family = FAMILIES.get(int(r.variant))
    if 5 <= int(r.variant) <= 11:  # patched-immediate kernels: SASS of the embedded cubin, placeholders in place
        kind = int(r.variant) - 4
        sym, sha = imm_symbol(L, kind), imm_sass_sha256(L, kind)
    else:
        sym = kernel_symbol(lib_path, family, L) if family else None
        sha = sass_sha256(lib_path, sym) if sym else None
    rec = kernel_record(sha)
    ipc, ipc_src = issue_peak_per_sm_clk()
    lanes, lanes_src = fp32_lane_peak_per_sm_clk()
    issue_peak = ipc * sm_count * sm_hz  # warp-instructions / s
    nominal_peak = lanes * sm_count * sm_hz
    nominal_achieved = per_launch_states * (n + 1) / search_s
    out = {"bound": "alu-issue", "unit": "Gwarp-instr/s", "achieved": None, "peak": issue_peak / 1e9, "frac": None,
           "traffic": None, "kernel": sym, "sass_sha256": sha, "search_ms_per_launch": search_s * 1e3,
           "peak_basis": f"{ipc:.3f} warp-instr/SM/clk {ipc_src} x {sm_count} SMs x {sm_hz / 1e6:.0f} MHz "
                         "(SM clock sampled during the timed region)",
           "nominal_frac": nominal_achieved / nominal_peak,
           "nominal_basis": f"{n + 1} ops/state (SURVEY.md §8d: n-1 field adds + 1 value add + 1 min) vs "
                            f"{lanes:.1f} FP32 lanes/SM/clk ({lanes_src}); > 1 = the table method's algorithmic saving"}
    if rec is None:
        out["note"] = ("no ncu record for this kernel's SASS in profiles/kernel_records.json (kernel changed "
                       "since the last capture): issue figures withheld")
        return out
    ips = float(rec["thread_instr_per_state"])
    achieved = per_launch_states * ips / 32.0 / search_s
    out.update({"achieved": achieved / 1e9, "frac": achieved / issue_peak, "instr_per_state": ips,
                "traffic": rec.get("dram_bytes_per_launch"),
                "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum of the ncu --set full capture "
                                f"({rec.get('capture')}); algorithmic HBM bytes per state: 0",
                "record": {k: rec.get(k) for k in ("capture", "issue_active_pct", "states", "workload")}})
    return out


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="E", choices=sorted(CONFIG_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the informational A-D config lines")
    ap.add_argument("--shared-device", action="store_true",
                    help="functional test of the N>1 path on fewer GPUs: ranks share devices, gloo collective "
                         "(not a scaling measurement)")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        clk = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        loaded = [c for c in clk if c > 500] or clk
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def dist_setup(gpus: int):
    """One process per GPU (torchrun).  QB_DIST_BACKEND=gloo forces the CPU collective, which lets
    several ranks share one GPU for a functional test of the N>1 path (their shard kernels are
    independent; the only exchange is the host-side all-reduce)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch

    if torch.cuda.is_available() and local >= torch.cuda.device_count():
        if not os.environ.get("QB_SHARED_DEVICE"):
            sys.exit(f"bench.py: rank {rank} has LOCAL_RANK {local} but only {torch.cuda.device_count()} CUDA "
                     "device(s) are visible (use --shared-device for a functional run on fewer GPUs)")
        local = local % torch.cuda.device_count()
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("QB_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def cpu_sample(coeffs, seconds: float):
    """Time the oracle port (reference solve_parallel restated in C, all host threads) on whole
    m-bit subspaces of the workload until ~`seconds` of CPU work; returns states/s."""
    from oracle import oracle

    n = coeffs.shape[0]
    threads = os.cpu_count() or 1
    m = max(0, n - 26)  # 2^26-state subspaces (solve_subspace granularity, SPEC.md §3.1)
    per_sub = 1 << (n - m)
    count = max(threads, 1)
    count = min(count, 1 << m)
    t0 = time.perf_counter()
    oracle.solve_subspaces(coeffs, m, 0, count, threads=threads)
    dt = time.perf_counter() - t0
    # grow to the target duration (whole subspaces, equal-sized, so states/s is unbiased)
    if dt < seconds and count < (1 << m):
        count2 = min(1 << m, max(count, int(count * seconds / max(dt, 1e-3))))
        count2 = max(threads, (count2 // threads) * threads)
        t0 = time.perf_counter()
        oracle.solve_subspaces(coeffs, m, 0, count2, threads=threads)
        dt = time.perf_counter() - t0
        count = count2
    states = count * per_sub
    return {"value": states / dt, "unit": "states/s", "cores": threads, "kind": "port",
            "sample": f"extrapolated from {count} of {1 << m} m={m} subspaces ({states:.3g} states, {dt:.1f} s) of config E via "
                      f"oracle/gray_oracle.c oc_solve_subspaces (reference solve_parallel restated), {threads} threads",
            "seconds": dt}


def numba_reference_sample(coeffs, seconds: float):
    """The UNMODIFIED reference package (baseline/_ref, staged by tools/stage_reference.sh; numba kernels) on the
    same kind of sample as cpu_sample: whole 2^26-state subspaces through its own ``solve_subspace`` on a thread pool
    of all host cores, which is what its ``solve_parallel`` runs (solver.py:214-222).  Informational: the arm's value
    stays the C port.  None / {"unavailable": ...} when the staged reference or numba is missing."""
    ref = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "qubrute")):
        return {"unavailable": "baseline/_ref/qubrute not staged (tools/stage_reference.sh)"}
    sys.path.insert(0, ref)
    try:
        import qubrute as ref_qb
        from concurrent.futures import ThreadPoolExecutor
    except Exception as exc:  # numba missing or broken
        return {"unavailable": f"{type(exc).__name__}: {exc}"}
    finally:
        sys.path.remove(ref)
    n = coeffs.shape[0]
    threads = os.cpu_count() or 1
    m = max(0, n - 26)
    inst = ref_qb.QuboInstance(coeffs)
    ref_qb.solve_incremental(ref_qb.random_instance(6, 0))  # JIT warm-up, as the reference's own bench does (cli.py:78-83)
    t0 = time.perf_counter()
    ref_qb.solve_subspace(inst, ref_qb.SubspaceSpec(m=m, suffix=0))
    one = time.perf_counter() - t0
    count = min(1 << m, threads * max(1, int(seconds / max(one, 1e-3))))
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(lambda sfx: ref_qb.solve_subspace(inst, ref_qb.SubspaceSpec(m=m, suffix=sfx)), range(count)))
    dt = time.perf_counter() - t0
    states = count * (1 << (n - m))
    return {"value": states / dt, "unit": "states/s", "cores": threads, "kind": "reference",
            "sample": f"{count} of {1 << m} m={m} subspaces ({states:.3g} states, {dt:.1f} s) through the unmodified "
                      f"reference's solve_subspace (numba {_numba_version()}) on a pool of {threads} threads",
            "seconds": dt}


def _numba_version() -> str:
    try:
        import numba
        return numba.__version__
    except Exception:
        return "?"


def extra_configs(qb, _lib, instances, reps: int = 5):
    """Informational per-config throughput (rank 0, N=1): BASELINE configs A-D besides the
    headline E.  kernel = device time of the solve launches (library CUDA events); e2e = the
    public API call with host buffers (planning, H2D, kernels, D2H)."""
    import numpy as np

    out = {}
    for name in ("A", "B", "D"):
        c = instances.config_coeffs(name, 0)
        inst = qb.QuboInstance(c)
        n = inst.n
        for _ in range(2):
            qb.solve_incremental(inst)
        ks, es = [], []
        for _ in range(reps):
            r = _lib.solve(inst.coeffs)
            ks.append(r.kernel_ms)
            t0 = time.perf_counter()
            qb.solve_incremental(inst)
            es.append(time.perf_counter() - t0)
        km, em = float(np.median(ks)), float(np.median(es))
        out[name] = {"n": n, "kernel_ms": km, "states_per_s": 2 ** n / (km * 1e-3), "e2e_ms": em * 1e3,
                     "e2e_states_per_s": 2 ** n / em, "exact_path": bool(r.exact)}
    batch = instances.config_batch(4096, 16)
    for _ in range(2):
        _lib.solve_batch(batch)
    ks, es = [], []
    for _ in range(reps):
        _, _, km = _lib.solve_batch(batch)
        ks.append(km)
        t0 = time.perf_counter()
        qb.solve_batch(batch, as_arrays=True)
        es.append(time.perf_counter() - t0)
    km, em = float(np.median(ks)), float(np.median(es))
    states = 4096 * 2 ** 16
    # the host folds + packs each instance's upper triangle (fp32 when exact, as for these fp32 draws)
    packed = 4096 * (16 * 17 // 2) * (4 if np.array_equal(batch.astype(np.float32), batch) else 8)
    out["C"] = {"n": 16, "instances": 4096, "kernel_ms": km, "states_per_s": states / (km * 1e-3),
                "e2e_ms": em * 1e3, "e2e_states_per_s": states / em, "h2d_bytes": int(packed),
                "note": "kernel_ms = device window of the 4 pipelined batch pieces (two compute streams); "
                        "e2e = solve_batch on the (4096,16,16) fp64 host array: host fold/pack on all "
                        "cores, pinned H2D per piece, kernels, one D2H"}
    return out


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU solver on the box's host cores.  When the unmodified reference is staged
    (baseline/_ref, numba importable) every step times IT (kind "reference") and one sample of the oracle port is
    reported beside it; otherwise the steps time the port (kind "port")."""
    from paper_2310_19373_b200 import instances

    if rank != 0:
        return
    coeffs = instances.config_coeffs(args.config, 0)
    n = coeffs.shape[0]
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    try:
        probe = numba_reference_sample(coeffs, 0.5)  # also the JIT warm-up
    except Exception as exc:
        probe = {"unavailable": f"{type(exc).__name__}: {exc}"}
    real = "value" in probe
    sample = (lambda sec: numba_reference_sample(coeffs, sec)) if real else (lambda sec: cpu_sample(coeffs, sec))
    for _ in range(args.warmup):
        sample(0.5)
    vals, secs = [], []
    for _ in range(args.steps):
        s = sample(per_step)
        vals.append(s["value"])
        secs.append(s["seconds"])
    value = statistics.median(vals)
    what = ("the unmodified reference package (baseline/_ref, numba kernels; solve_subspace on a thread pool, as its "
            "solve_parallel runs)" if real else "oracle/gray_oracle.c (the reference's solve_parallel restated in C)")
    line = {
        "impl": "reference", "metric": "QUBO states evaluated/sec (2^n / solve time)", "value": value,
        "unit": "states/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64, bench_seed(40,0))",
        "extrapolated": True,
        "extrapolation": f"each step times a bounded sample of {what} ({s['sample']}, median "
                         f"{statistics.median(secs):.1f} s); "
                         f"value = sampled states/s (subspaces are equal-sized, so the rate is unbiased); "
                         "ms_per_step = the timed sample; full_solve_ms_extrapolated = 2^n states at that rate",
        "full_solve_ms_extrapolated": 1e3 * 2 ** n / value,
        "config": bench_config(args.config, n),
        "cpu_baseline": {"value": value, "unit": "states/s", "cores": s["cores"], "kind": s["kind"],
                         "sample": s["sample"]},
        "e2e": {"value": value, "unit": "states/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if real:
        # the C port beside the real reference, one sample (the GPU arm's cpu_baseline uses the port)
        port = cpu_sample(coeffs, min(per_step, 10.0))
        line["oracle_port"] = {k: port[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line["oracle_port"]["port_over_reference"] = port["value"] / value
    else:
        line["reference_numba"] = probe
    print(json.dumps(line), flush=True)


def bench_config(name: str, n: int) -> dict:
    """The workload description, identical in both arms (the driver compares them)."""
    return {"workload": CONFIG_DESC[name], "n": n, "states_per_solve": 2 ** n,
            "l2": "GPU arm: 256 MiB buffer written between timed steps (> 126 MB L2); CPU arm: host caches, no flush"}


def self_launch(args) -> None:
    """``--gpus N`` (N > 1) outside torchrun: re-launch this command as N ranks (one per GPU, NCCL,
    127.0.0.1 rendezvous) -- the driver's torchrun form -- after checking that N devices exist."""
    import socket

    import torch

    have = torch.cuda.device_count()
    env = dict(os.environ)
    if have < args.gpus:
        if not args.shared_device:
            sys.exit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible; a multi-GPU number needs "
                     f"{args.gpus} GPUs (--shared-device runs the {args.gpus} ranks on the visible devices over "
                     "gloo as a functional test, not a scaling measurement)")
    if args.shared_device:
        env["QB_SHARED_DEVICE"] = "1"
        env["QB_DIST_BACKEND"] = "gloo"
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator lines show nranks = N
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=env))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        self_launch(args)
    if args.shared_device:
        os.environ["QB_SHARED_DEVICE"] = "1"
        os.environ.setdefault("QB_DIST_BACKEND", "gloo")
    if args.impl == "reference":
        # CPU only, rank 0 alone: no process group, no collective (the other ranks of a torchrun launch exit 0)
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup(args.gpus)
    os.environ["QB_DEVICE"] = str(local)  # the library's default device follows the rank -> GPU map

    import numpy as np
    import torch

    import paper_2310_19373_b200 as qb
    from paper_2310_19373_b200 import _lib, distributed, instances

    torch.cuda.set_device(local)
    _lib.init(local)
    coeffs = instances.config_coeffs(args.config, 0)
    inst = qb.QuboInstance(coeffs)
    n = inst.n
    states = 2 ** n
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    coll_dev = "cuda" if world == 1 or torch.distributed.get_backend() == "nccl" else "cpu"

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def device_step():
        res = _lib.solve(inst.coeffs, 0, 0, 0, _lib.TIE_GRAY, shard=rank, shard_count=world, variant=args.variant)
        if world > 1:
            distributed.allreduce_argmin(res)
        return res

    warm = [device_step() for _ in range(args.warmup)]
    module_ms = max(float(w.module_ms) for w in warm) if warm else 0.0
    barrier()

    # ---- device-time measurement (value)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.25)
    kernel_ms, search_ms, launches, results = 0.0, 0.0, 0, []
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        r = device_step()
        kernel_ms += r.kernel_ms
        search_ms += r.search_ms
        launches += r.launches
        results.append(r)
    barrier()
    kernel_ms_max = max_over_ranks(kernel_ms)
    search_ms_max = max_over_ranks(search_ms)

    # ---- end-to-end through the public API (e2e)
    e2e_s = 0.0
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        t0 = time.perf_counter()
        if world == 1:
            sol = qb.solve_incremental(inst)
        else:
            sol = distributed.solve_sharded(inst)
        e2e_s += time.perf_counter() - t0
    barrier()
    e2e_max = max_over_ranks(e2e_s)
    clocks = sampler.stop()
    # cold path, reported beside e2e (not a timed step): the first solve of a table this process has not
    # seen, i.e. including the patched-immediate module build + load (config E, seed rep 1)
    cold_ms = None
    if world == 1:
        cold_inst = qb.QuboInstance(instances.config_coeffs(args.config, 1))
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        qb.solve_incremental(cold_inst)
        cold_ms = 1e3 * (time.perf_counter() - t0)

    r = results[-1]
    value = states * args.steps / (kernel_ms_max * 1e-3)
    e2e_value = states * args.steps / e2e_max
    # roofline of the dominant (search) kernel: per-GPU launch = states/world states
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    sm_hz = (clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0) * 1e6
    per_launch_states = states / world
    search_s = search_ms_max * 1e-3 / args.steps
    roofline = roofline_block(r, n, per_launch_states, search_s, sm_count, sm_hz, _lib.LIB_PATH)
    d2h = 48 + 8 + 8 * int(r.candidates) if not r.exact else 48
    line = {
        "metric": "QUBO states evaluated/sec (2^n / solve time)",
        "value": value, "unit": "states/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": kernel_ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded splitmix64 + Box-Muller, bench_seed(40,0); BASELINE config E)",
        "config": bench_config(args.config, n),
        "geometry": {"shards": world, "parallelism": f"prefix-shard x{world}", "prefix_bits": int(r.prefix_bits),
                     "exact_path": bool(r.exact), "scale_exp": int(r.scale_exp), "candidates": int(r.candidates),
                     "exact_blocks": int(r.exact_blocks), "blocks": int(per_launch_states) >> 10,
                     "auto_retries": int(r.retries),
                     "argmin": hex(qb.bits_to_int(sol.minimizer)), "min_value": sol.value},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": "states/s", "h2d_bytes_per_step": int(r.param_bytes) * int(r.launches),
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_max * 1e3 / args.steps},
        "gpu_launches": launches,
        "imm_module": {"load_ms": module_ms, "e2e_first_solve_of_new_table_ms": cold_ms,
                       "note": "the patched-immediate search kernel (QB_VARIANT_IMM*) is built for an instance by "
                               "writing its coarse table into a cubin copy and loading it (first solve of a table, "
                               "in the warm-up here); later solves of the same table reuse the loaded module, as "
                               "the timed value and e2e steps do"},
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_extra:
        line["configs"] = extra_configs(qb, _lib, instances)
        # the other traversal kernels on the same workload: the table-load coarse kernel, the fp32 table
        # kernel and the literal per-step field walk (QB_VARIANT_COARSE / _TABLE / _FIELDWALK)
        names = {0: "auto", 1: "table", 2: "fieldwalk", 3: "coarse_tableload", 4: "tc", 5: "coarse_imm",
                 6: "coarse_imm_superblock", 7: "threshold_imm8", 8: "threshold_imm8_superblock", 9: "threshold_imm8_rowbound",
                 10: "threshold_imm8_rowbound_superblock", 11: "threshold_imm8_rowbound_12bit",
                 12: "threshold_byte8_tableload"}
        line["variants"] = {f"{names[int(r.variant)]} (default)": {
            "search_ms": search_s * 1e3, "states_per_s": per_launch_states / search_s}}
        # (the tensor-core pass, QB_VARIANT_TC, is retired from this list: 40 ms, TMEM round-trip bound,
        # DESIGN.md section 4)
        for var in (_lib.VARIANT_BYTE8, _lib.VARIANT_IMM8AQ, _lib.VARIANT_IMM8AS, _lib.VARIANT_IMM8A, _lib.VARIANT_IMM8S, _lib.VARIANT_IMM8, _lib.VARIANT_IMM, _lib.VARIANT_COARSE, _lib.VARIANT_TABLE,
                    _lib.VARIANT_FIELDWALK):
            _lib.solve(inst.coeffs, variant=var)
            vr = _lib.solve(inst.coeffs, variant=var)
            vs = states / (vr.search_ms * 1e-3)
            line["variants"][names[int(vr.variant)]] = {"search_ms": vr.search_ms, "states_per_s": vs,
                                           "nominal_frac": roofline["nominal_frac"] * vs / (per_launch_states / search_s),
                                           "same_argmin": int(vr.argmin_bits) == int(r.argmin_bits)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the unmodified reference (numba, baseline/_ref) when it is staged -- on the GPU boxes it is about twice as
        # fast as the C port (r15: 1.12e9 against 5.3e8 states/s on 16 threads) -- else the port; the port is kept beside it
        port = cpu_sample(inst.coeffs, args.cpu_seconds)
        port.pop("seconds", None)
        try:
            real = numba_reference_sample(np.asarray(inst.coeffs, dtype=np.float64), args.cpu_seconds)
        except Exception as exc:
            real = {"unavailable": f"{type(exc).__name__}: {exc}"}
        if "value" in real:
            real.pop("seconds", None)
            line["cpu_baseline"] = real
            line["cpu_baseline_port"] = port
        else:
            line["cpu_baseline"] = port
            line["cpu_baseline_reference"] = real
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
