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
sampled during the timed region.  cpu_baseline: the oracle port of the reference's solver
(oracle/, C, all host threads) on a bounded sample of the same workload, rank 0 at N=1.
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
# FP32 add-lane peak: measured on this pool's B200 by tools/alu_peaks.cu (profiles/r01_alu_peaks.json,
# CUDA events, 2 CTAs x 512 threads/SM); fallback = 128 lanes/SM/clk x SMs x max SM clock
ALU_PEAKS = os.path.join(ROOT, "profiles", "r01_alu_peaks.json")
FP32_ADD_LANES_PER_SM_CLK = 128.0
ISSUE_WARP_INSTR_PER_SM_CLK = 4.0
# ncu --set full capture of the search kernel (DRAM bytes per launch, n=40 config E)
NCU_SUMMARY = os.path.join(ROOT, "profiles", "r11_ncu_search_summary.txt")


def ncu_traffic_bytes():
    """dram__bytes_read.sum + dram__bytes_write.sum of the committed capture, in bytes, or None."""
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        vals = {}
        with open(NCU_SUMMARY) as fh:
            for line in fh:
                if line.startswith("dram__bytes_read.sum =") or line.startswith("dram__bytes_write.sum ="):
                    k, rest = line.split("=")
                    num, unit = rest.split()
                    vals[k.strip()] = float(num) * scale[unit]
        return vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    except (OSError, KeyError, ValueError):
        return None


# SASS instructions per state of the table kernel's inner block (cuobjdump count)
SASS_INSTR_PER_STATE = 1.032  # ncu smsp__inst_executed x 32 / 2^40 of the coarse kernel (profiles/r11_ncu_search_summary.txt)


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

    if torch.cuda.is_available():
        local = local % max(1, torch.cuda.device_count())
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
            "sample": f"{count} of {1 << m} m={m} subspaces ({states:.3g} states, {dt:.1f} s) of config E via "
                      f"oracle/gray_oracle.c oc_solve_subspaces (reference solve_parallel restated), {threads} threads",
            "seconds": dt}


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
    out["C"] = {"n": 16, "instances": 4096, "kernel_ms": km, "states_per_s": states / (km * 1e-3),
                "e2e_ms": em * 1e3, "e2e_states_per_s": states / em,
                "h2d_bytes": int(batch.nbytes)}
    return out


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU solver (oracle port) on the box's host cores."""
    from paper_2310_19373_b200 import instances

    if rank != 0:
        return
    coeffs = instances.config_coeffs(args.config, 0)
    n = coeffs.shape[0]
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_sample(coeffs, 0.5)
    vals, secs = [], []
    for _ in range(args.steps):
        s = cpu_sample(coeffs, per_step)
        vals.append(s["value"])
        secs.append(s["seconds"])
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "QUBO states evaluated/sec (2^n / solve time)", "value": value,
        "unit": "states/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64, bench_seed(40,0))",
        "config": {"workload": CONFIG_DESC[args.config], "n": n, "states_per_solve": 2 ** n},
        "cpu_baseline": {"value": value, "unit": "states/s", "cores": s["cores"], "kind": "port",
                         "sample": s["sample"]},
        "e2e": {"value": value, "unit": "states/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_setup(args.gpus)
    os.environ["QB_DEVICE"] = str(local)  # the library's default device follows the rank -> GPU map
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

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

    for _ in range(args.warmup):
        device_step()
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

    r = results[-1]
    value = states * args.steps / (kernel_ms_max * 1e-3)
    e2e_value = states * args.steps / e2e_max
    # roofline of the dominant (search) kernel: per-GPU launch = states/world states
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    sm_hz = (clocks.get("sm_max_mhz") or 1965.0) * 1e6
    per_launch_states = states / world
    search_s = search_ms_max * 1e-3 / args.steps
    achieved = per_launch_states * (n + 1) / search_s
    peak = FP32_ADD_LANES_PER_SM_CLK * sm_count * sm_hz
    peak_src = "fallback 128 lanes/SM/clk x SMs x max SM clock"
    try:
        with open(ALU_PEAKS) as fh:
            peak = float(json.load(fh)["results"]["fadd2"]["lane_ops_per_s"])
        peak_src = "measured FP32 add-lane rate (tools/alu_peaks.cu, profiles/r01_alu_peaks.json)"
    except (OSError, KeyError, ValueError):
        pass
    issue_peak = ISSUE_WARP_INSTR_PER_SM_CLK * 32 * sm_count * sm_hz
    roofline = {
        "bound": "alu", "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "Gop/s",
        "frac": achieved / peak, "traffic": ncu_traffic_bytes(),
        "traffic_note": f"DRAM bytes per search launch from the committed ncu capture ({os.path.relpath(NCU_SUMMARY, ROOT)}, "
                        "n=40): the per-chunk minima and CTA records; the algorithmic HBM traffic per state is 0",
        "basis": f"nominal {n + 1} ops/state (SURVEY.md §8d: n-1 field adds + 1 value add + 1 min) vs the "
                 f"{peak_src}; the coarse kernel issues ~{SASS_INSTR_PER_STATE} SASS instr/state, so frac > 1 "
                 "measures the algorithmic saving and issue_frac (vs 4 warp-instr/SM/clk) the kernel quality",
        "issue_frac": per_launch_states * SASS_INSTR_PER_STATE / search_s / issue_peak,
        "search_ms_per_launch": search_s * 1e3,
    }
    d2h = 48 + 8 + 8 * int(r.candidates) if not r.exact else 48
    line = {
        "metric": "QUBO states evaluated/sec (2^n / solve time)",
        "value": value, "unit": "states/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": kernel_ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded splitmix64 + Box-Muller, bench_seed(40,0); BASELINE config E)",
        "config": {"workload": CONFIG_DESC[args.config], "n": n, "states_per_solve": states,
                   "shards": world, "prefix_bits": int(r.prefix_bits), "exact_path": bool(r.exact),
                   "scale_exp": int(r.scale_exp), "candidates": int(r.candidates),
                   "l2": "256 MiB buffer written between timed steps",
                   "argmin": hex(qb.bits_to_int(sol.minimizer)),
                   "min_value": sol.value, "parallelism": f"prefix-shard x{world}"},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": "states/s", "h2d_bytes_per_step": int(r.param_bytes) * int(r.launches),
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_max * 1e3 / args.steps},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_extra:
        line["configs"] = extra_configs(qb, _lib, instances)
        # the other traversal kernels on the same workload: the fp32 table kernel, the literal
        # per-step field walk and the tensor-core coarse pass (QB_VARIANT_TABLE / _FIELDWALK / _TC)
        names = {0: "auto", 1: "table", 2: "fieldwalk", 3: "coarse", 4: "tc"}
        line["variants"] = {f"{names[int(r.variant)]} (default)": {
            "search_ms": search_s * 1e3, "states_per_s": per_launch_states / search_s}}
        for var in (_lib.VARIANT_TABLE, _lib.VARIANT_FIELDWALK, _lib.VARIANT_TC):
            _lib.solve(inst.coeffs, variant=var)
            vr = _lib.solve(inst.coeffs, variant=var)
            vs = states / (vr.search_ms * 1e-3)
            line["variants"][names[int(vr.variant)]] = {"search_ms": vr.search_ms, "states_per_s": vs,
                                           "nominal_roofline_frac": vs * (n + 1) / peak,
                                           "same_argmin": int(vr.argmin_bits) == int(r.argmin_bits)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_sample(inst.coeffs, args.cpu_seconds)
        cb.pop("seconds", None)
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
