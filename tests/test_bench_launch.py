"""bench.py launch plumbing on CPU: `--gpus N` re-launches itself under torchrun (one
process per GPU, 127.0.0.1 rendezvous) and every rank reaches the multi-rank arm."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(out: str) -> dict:
    rows = [r for r in out.splitlines() if r.startswith("{")]
    assert rows, out
    return json.loads(rows[-1])


@pytest.mark.parametrize("n,entry", [(1, "run_ours"), (2, "run_ours_dist")])
def test_bench_gpus_n_reaches_the_arm(n, entry):
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(n),
                        "--dry-run"], capture_output=True, text=True, env=env, timeout=240)
    assert p.returncode == 0, p.stderr[-3000:]
    d = _line(p.stdout)
    assert d["entry"] == entry and d["n_gpus"] == n
    if n > 1:
        assert d["rank_sum"] == n * (n - 1) / 2
