"""bench.py's own N-rank launch on CPU: ``--gpus 2 --dry-run`` re-executes
itself under torch.distributed.run (gloo, 127.0.0.1), every rank runs the
sharded host protocol (chained einsum-order norm pass over its row shard,
redundant draws) and rank 0 reports that the ranks agree bit for bit and
equal the single-process numpy norms."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("ranks", [1, 2, 3])
def test_bench_dry_run_ranks_agree(ranks):
    env = dict(os.environ, PYTHONPATH=ROOT, OMP_NUM_THREADS="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(ranks),
                        "--dry-run"], capture_output=True, text=True, timeout=600, env=env,
                       cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    out = json.loads(lines[0])
    assert out["dry_run"] and out["n_ranks"] == ranks
    assert out["agree"] and out["norms_equal_numpy"]
    assert out["rounds"] > 1
