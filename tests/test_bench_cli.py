"""bench.py's multi-GPU entry point (VERDICT r1 "make SCALE measurable").

* CPU: ``bench.py --gpus 2`` outside torchrun with fewer than 2 visible GPUs fails loudly instead
  of timing one GPU and calling it a 2-GPU number.
* GPU: ``bench.py --gpus 2 --shared-device`` re-launches itself as 2 torchrun ranks (gloo
  collective, both shards on the one visible B200): the N>1 code path end to end, with the same
  argmin as the 1-rank run.  Its time is two shards contending for one GPU, not a scaling number.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _bench(*args, timeout=900):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_gpus_without_devices_fails_loudly():
    import torch

    have = torch.cuda.device_count()
    r = _bench("--gpus", str(max(2, have + 1)), "--steps", "1", "--warmup", "3")
    assert r.returncode != 0
    assert f"only {have} CUDA device(s) visible" in r.stderr


@pytest.mark.gpu
def test_shared_device_two_ranks_runs_the_sharded_path():
    common = ["--steps", "1", "--warmup", "3", "--config", "D", "--no-extra", "--no-cpu-baseline"]
    one = _bench("--gpus", "1", *common)
    assert one.returncode == 0, one.stderr[-3000:]
    two = _bench("--gpus", "2", "--shared-device", *common)
    assert two.returncode == 0, two.stderr[-3000:]
    l1 = json.loads(one.stdout.strip().splitlines()[-1])
    l2 = json.loads(two.stdout.strip().splitlines()[-1])
    assert l2["n_gpus"] == 2 and l2["geometry"]["shards"] == 2
    assert l2["geometry"]["argmin"] == l1["geometry"]["argmin"]
    assert l2["geometry"]["min_value"] == l1["geometry"]["min_value"]
