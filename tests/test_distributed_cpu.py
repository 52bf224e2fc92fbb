"""Multi-rank path on CPU (gloo, world_size 2 and 3): the shard combine and the single
all-reduce(MIN) exchange of distributed.solve_sharded.

The per-rank GPU solve is replaced by an injected CPU shard solver (numpy enumeration
from the oracle) that splits the state space the same way (equal contiguous slices of
the chunk space) and reports (value_key, tie_key, argmin) like qb_solve; everything
above it — packing, the collective, the lexicographic pick — is the product code.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _Res:
    pass


def _ordered(v: float) -> int:
    import struct

    if v == 0.0:
        v = 0.0
    b = struct.unpack("<Q", struct.pack("<d", v))[0]
    return (~b & 0xFFFFFFFFFFFFFFFF) if b >> 63 else (b | (1 << 63))


def make_cpu_shard_solver(k: int):
    """qb_solve stand-in: shard `shard` of `shard_count` equal slices of the 2^k chunk prefixes."""

    def solve_fn(coeffs, m_fix, suffix, m_tie, rule, shard=0, shard_count=1):
        n = coeffs.shape[0]
        vals = O.all_values(coeffs)
        keys = O.tie_keys(n, m_tie)
        chunks = 1 << k
        cb, ce = chunks * shard // shard_count, chunks * (shard + 1) // shard_count
        r = _Res()
        r.states = (ce - cb) << (n - k)
        if ce == cb:
            r.value_key = r.tie_key = (1 << 64) - 1
            r.argmin_bits = 0
            return r
        lo, hi = cb << (n - k), ce << (n - k)
        xs = np.arange(lo, hi, dtype=np.int64)
        v = vals[lo:hi]
        vmin = v.min()
        cand = xs[v == vmin]
        best = cand[np.argmin(keys[cand])]
        r.value_key = _ordered(float(vmin))
        r.tie_key = int(keys[best])
        r.argmin_bits = int(best)
        return r

    return solve_fn


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2310_19373_b200 as qb
    from paper_2310_19373_b200 import distributed

    out = []
    for coeffs, mode, m, k in cases:
        inst = qb.QuboInstance(coeffs)
        cfg = qb.SolveConfig(threads=2, fixed_bits=m) if mode == "parallel" else None
        sol = distributed.solve_sharded(inst, mode=mode, config=cfg, solve_fn=make_cpu_shard_solver(k))
        out.append((qb.bits_to_int(sol.minimizer), sol.value, sol.evaluations))
    q.put((rank, out))
    dist.destroy_process_group()


def _run(world, cases):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_solve_combines_like_single_solve(world):
    from paper_2310_19373_b200 import instances

    cases = []
    for rep in range(3):
        cases.append((instances.int_uniform_coeffs(10, 900 + rep, -2, 2), "incremental", 0, 4))  # ties
        cases.append((instances.config_coeffs("E", rep, n=12), "incremental", 0, 5))
        cases.append((instances.int_uniform_coeffs(9, 950 + rep, -1, 1), "parallel", 3, 3))
    cases.append((np.zeros((8, 8)), "incremental", 0, 3))  # every state tied
    res = _run(world, cases)
    for r in range(world):
        assert res[r] == res[0]  # every rank returns the same answer
    for (coeffs, mode, m, k), (bits, value, evals) in zip(cases, res[0]):
        want_bits, want_val, _ = O.expected_argmin(coeffs, m)
        assert bits == want_bits
        assert value == O.eval_upper(coeffs, [(bits >> i) & 1 for i in range(coeffs.shape[0])])
        n = coeffs.shape[0]
        assert evals == ((1 << n) - (1 << m) if mode == "parallel" else (1 << n) - 1)


def test_combine_skips_empty_shards():
    from paper_2310_19373_b200.distributed import INT64_MAX, combine_shards

    rows = [INT64_MAX, 5, 5, INT64_MAX, 9, 3, 0, 17, 11]  # world 3: vk | tk | x
    assert combine_shards(rows, 3) == (5, 3, 11)
