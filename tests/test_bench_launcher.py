"""bench.py's multi-GPU launcher on CPU (no GPU needed): `--gpus 2 --dry-run`
re-launches itself under torch.distributed.run with 2 ranks (gloo, 127.0.0.1),
every rank takes its cyclic tile-row share of the C5 triangle (mds_plan), and
rank 0 prints one JSON line: the shares partition the N(N-1)/2 pairs and are
balanced (within ~1% at N = 100k)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("gpus,workload", [(2, "C5"), (3, "C4")])
def test_bench_launcher_dry_run(gpus, workload):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--dry-run",
                        "--workload", workload], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["dry_run"] and out["n_gpus"] == gpus
    assert len(out["pairs_per_rank"]) == gpus
    assert out["total_pairs"] == out["expected_pairs"]
    assert out["balance_max_over_mean"] < 1.02
