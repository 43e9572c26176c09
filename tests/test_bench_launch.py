"""bench.py's multi-GPU launcher on CPU: `--gpus N` outside torchrun re-launches itself as N
ranks (torch.distributed.run, 127.0.0.1); `--dry-run` runs the sharded orchestration over
gloo with the numpy test ops and prints one JSON line with n_gpus = N. Without N visible
GPUs a real run fails loudly instead of measuring fewer."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    return p


@pytest.mark.parametrize("n,config,scaling", [(2, "cfg3", "weak"), (3, "cfg5", "strong")])
def test_dry_run_launches_n_ranks(n, config, scaling):
    p = _run("--gpus", str(n), "--dry-run", "--config", config)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == n and line["dry_run"] and line["scaling"] == scaling
    assert line["parity"] == "bit-exact vs the C oracle"
    assert sum(f"rank {r}/{n}" in p.stderr for r in range(n)) == n


def test_real_run_without_gpus_fails_loudly():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("GPUs visible")
    p = _run("--gpus", "2", "--steps", "1", timeout=300)
    assert p.returncode != 0 and "CUDA device" in (p.stderr + p.stdout)
