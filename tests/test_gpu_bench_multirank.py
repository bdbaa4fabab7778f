"""bench.py --gpus N end to end: without torchrun it re-launches itself
under torch.distributed.run; each rank owns E global env ids; the per-env stats and
state checksums are all-gathered at the end.  Here two ranks share the one GPU over
gloo (their kernels never wait on each other -- the only exchange is the final
gather), and the checksum over the first E global envs must equal the N=1 run's."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--envs", "64", "--steps", "10", "--warmup", "3", "--no-cpu-baseline", "--no-step-batch",
        "--sample-reps", "1", "--sync-steps", "2", "--e2e-steps", "2", "--phase-steps", "2", "--backend", "gloo"]


def _bench(gpus):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus)] + ARGS,
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_two_ranks_match_one(torch_cuda):
    two = _bench(2)
    one = _bench(1)
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["stats"]["envs"] == 128 and two["stats"]["comm_nranks_ok"]
    assert two["stats"]["state_checksum_first_envs"] == one["stats"]["state_checksum_first_envs"]
    assert two["stats"]["state_checksum"] != two["stats"]["state_checksum_first_envs"]
    assert two["value"] > 0 and two["e2e"]["value"] > 0
