"""bench.py's launch contract on a host without enough GPUs: `--gpus N` outside torchrun re-launches itself as N
ranks only if the box has N GPUs, and otherwise fails with a one-line JSON error (no silent single-rank run);
under torchrun, --gpus must equal WORLD_SIZE."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(torch.cuda.device_count() >= 2, reason="the box has 2 GPUs: bench.py would launch 2 ranks")
def test_gpus_2_without_two_gpus_fails_clearly():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], capture_output=True, text=True,
                       timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" in line and "2 GPUs" in line["error"]


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True, text=True,
                       timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in json.loads(r.stdout.strip().splitlines()[-1])["error"]
