"""bench.py's launcher on CPU (no GPU work): --gpus N without a torchrun environment
launches N ranks itself (torch.distributed.run on 127.0.0.1), each rank gets its
placement; --gpus disagreeing with WORLD_SIZE fails loudly."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, cwd=ROOT, env=e)


def test_gpus_flag_launches_ranks_block_placement():
    r = _bench("--gpus", "2", "--config", "C4", "--dry-run")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 and d["placement"] == "block" for d in lines)
    got = {d["rank"]: [tuple(b) for b in d["blocks"]] for d in lines}
    # configs[3]: 8 feature blocks of one node, contiguous halves per GPU
    assert got[0] == [(0, j) for j in range(4)] and got[1] == [(0, j) for j in range(4, 8)]


def test_gpus_flag_node_placement_default():
    r = _bench("--gpus", "2", "--dry-run")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    got = {d["rank"]: [tuple(b) for b in d["blocks"]] for d in lines}
    assert got[0] == [(i, 0) for i in range(4)] and got[1] == [(i, 0) for i in range(4, 8)]


def test_gpus_flag_mismatch_fails():
    r = _bench("--gpus", "2", "--config", "C1", env=dict(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
