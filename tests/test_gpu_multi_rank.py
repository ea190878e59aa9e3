"""The N>1 bench path on the device: `bench.py --gpus 2`
started outside any launcher re-executes itself as two ranks through the
same launcher entry the driver's torchrun uses (launch_local_ranks ->
torch.distributed.run, 127.0.0.1); each rank owns its own allocator and HBM
arena and runs the fused decode step with no collective on the hot path;
after the timed region rank 0 gathers sampled requests' outputs and layer
slices and checks them against the C oracle.  With one GPU both ranks share
it (gloo for the gather); the JSON line must say n_gpus = 2, verified."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def test_bench_two_ranks_verified():
    env = dict(os.environ, JENGA_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--batch-per-gpu", "4", "--ctx", "1536",
                        "--layers-per-group", "2", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 8
    assert d["verified"] is True and d["verification"]["samples"] == 4, d.get("verification")
    assert d["verification"]["max_rel_err"] <= 1e-2
