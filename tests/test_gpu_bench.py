"""bench.py plumbing on the GPU: `--gpus 2` launches itself as two ranks
(torch.distributed.run; gloo collectives so both ranks can share this box's
single GPU -- the driver's N-GPU runs use NCCL) and prints one JSON line with
n_gpus 2 whose assembled system is bitwise the one-GPU system."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _bench(*args, env=None):
    e = dict(os.environ, **(env or {}))
    e.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=900, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_gpus2_self_launch_bitwise_equals_one_gpu():
    common = ["--config", "C1", "--steps", "1", "--warmup", "1", "--verify", "--no-e2e",
              "--no-cpu-baseline"]
    one = _bench("--gpus", "1", *common)
    two = _bench("--gpus", "2", *common, env={"NLFEM_BENCH_BACKEND": "gloo"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["system_sha256"] == one["system_sha256"]
    assert two["element_pairs"] == one["element_pairs"]
    assert (two["mc_samples"], two["mc_hits"]) == (one["mc_samples"], one["mc_hits"])
    assert two["config"] == one["config"]
