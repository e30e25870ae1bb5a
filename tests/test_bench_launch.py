"""bench.py --gpus N without torchrun re-launches itself as N ranks (torch.distributed.run on
127.0.0.1); --launch-check makes the ranks meet over gloo, so this runs on CPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # one JSON line, from rank 0 only
    return json.loads(lines[0])


def test_gpus2_self_launches_two_ranks():
    d = _run("--gpus", "2", "--launch-check")
    assert d["world_size"] == 2 and d["ranks_seen"] == 2


def test_gpus1_stays_single_process():
    d = _run("--gpus", "1", "--launch-check")
    assert d["world_size"] == 1 and d["ranks_seen"] == 1
