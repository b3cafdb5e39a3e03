"""bench.py --gpus N outside torchrun launches N ranks itself (one process per
GPU, the driver's launch shape) and rank 0 prints one line; a --gpus that
disagrees with the launcher's world size fails loudly.  CPU only: the
CHESS_BENCH_PLUMBING skeleton (gloo process group, barrier, max over ranks)."""

import json
import os
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent


def _run(args, extra_env=None):
    env = {**os.environ, "CHESS_BENCH_PLUMBING": "1", **(extra_env or {})}
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        if not extra_env or k not in extra_env:
            env.pop(k, None)
    return subprocess.run([sys.executable, str(REPO / "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=240)


def test_gpus_two_spawns_two_ranks():
    r = _run(["--gpus", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["ranks"] == [0, 1] and out["max_over_ranks"] == 2.0


def test_gpus_mismatch_fails_loudly():
    r = _run(["--gpus", "4"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "--gpus 4" in r.stderr
