"""Multi-GPU solve: one process per GPU, the chunk space sharded across ranks.

Each rank scans an equal contiguous slice of the chunk (prefix) space on its own
device (qb_solve with shard=rank, shard_count=world), with no data-path
communication.  The only exchange is the final argmin: one all-reduce(MIN) over
a [3 * world] int64 buffer in which rank r fills slots r, world + r, 2*world + r
with its (value_key, tie_key, argmin) and every other slot is INT64_MAX, so the
MIN acts as an all-gather; every rank then picks the lexicographic minimum
(value_key, tie_key) locally.  Over NCCL this is one ~200-byte
collective on NVLink; under gloo (CPU tests) the same code path runs on CPU tensors.

The reference's counterpart is the ThreadPoolExecutor fan-out plus
combine_subspace_minima of solve_parallel (solver.py:193-229).
"""

from __future__ import annotations

import time

import numpy as np

from . import _lib
from .core import MAX_DIM, DimensionCapError, QuboInstance, bits_from_int
from .solver import Solution, SolveConfig, _resolve_m

_SIGN = 1 << 63
INT64_MAX = (1 << 63) - 1


def _to_i64(u: int) -> int:
    """Order-preserving map uint64 -> int64."""
    return int(u) - _SIGN


def combine_shards(rows, world: int):
    """Pick the winner from gathered [3*world] int64 slots (value_key, tie_key, argmin)."""
    best = None
    for r in range(world):
        vk, tk, x = int(rows[r]), int(rows[world + r]), int(rows[2 * world + r])
        if vk == INT64_MAX and tk == INT64_MAX:
            continue
        cand = (vk, tk, x)
        if best is None or cand[:2] < best[:2]:
            best = cand
    return best


def allreduce_argmin(res, group=None):
    """One all_reduce(MIN) exchanging every rank's (value_key, tie_key, argmin)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.full((3 * world,), INT64_MAX, dtype=torch.int64)
    buf[rank] = _to_i64(res.value_key)
    buf[world + rank] = _to_i64(res.tie_key)
    buf[2 * world + rank] = int(res.argmin_bits)
    buf = buf.to(device)
    dist.all_reduce(buf, op=dist.ReduceOp.MIN, group=group)
    rows = buf.cpu().tolist()
    return combine_shards(rows, world)


def solve_sharded(instance: QuboInstance, mode: str = "incremental", config: SolveConfig | None = None,
                  group=None, solve_fn=None) -> Solution:
    """Exhaustive solve of ``instance`` split across the ranks of ``group``.

    mode "incremental" (global Gray-rank ties) or "parallel" (``config.fixed_bits`` /
    ``threads`` tie rule, as solve_parallel).  Every rank returns the same Solution.
    ``solve_fn`` (default: the native qb_solve) is injectable so the host-side
    sharding/combine logic can be tested on CPU ranks.
    """
    import torch.distributed as dist

    if instance.n > MAX_DIM:
        raise DimensionCapError(f"n={instance.n} exceeds cap {MAX_DIM}")
    if mode == "parallel":
        m = _resolve_m(instance, config)
        evaluations = (1 << instance.n) - (1 << m)
    elif mode == "incremental":
        m = 0
        evaluations = (1 << instance.n) - 1
    else:
        raise ValueError(f"unsupported sharded mode {mode!r}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    solve_fn = solve_fn or _lib.solve
    t0 = time.perf_counter()
    res = solve_fn(instance.coeffs, 0, 0, m, _lib.TIE_GRAY, shard=rank, shard_count=world)
    best = allreduce_argmin(res, group)
    if best is None:
        raise RuntimeError("no shard produced a result")
    x = best[2]
    minimizer = bits_from_int(x, instance.n)
    value = _lib.eval_upper(instance.coeffs, minimizer.astype(np.float64))
    return Solution(minimizer=minimizer, value=value, evaluations=evaluations,
                    elapsed=max(time.perf_counter() - t0, 1e-9))
