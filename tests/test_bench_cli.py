"""CPU checks of bench.py's distributed harness:
`bench.py --gpus 2` without a torchrun environment re-launches itself as 2 ranks under
torch.distributed.run, and `--dry-run` runs the harness over gloo -- rendezvous, the
time-slab partition of every rank, the max-over-ranks reduction -- printing one JSON line
with n_gpus = 2 on rank 0 only."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("gpus", [2, 3])
def test_bench_gpus_respawns_and_prints_one_line(gpus):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--dry-run",
                          "--steps", "2"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    res = json.loads(lines[0])
    assert res["n_gpus"] == gpus and res["dry_run"] is True
    assert res["config"]["workload"] == "config4" and res["config"]["parallelism"] == f"time-slab x{gpus}"
    part = res["partition"]
    assert part["dofs_total"] == res["config"]["N"]
    n_t, Ns = res["config"]["n_t"], res["config"]["n_s"] ** res["config"]["d"]
    assert part["max_slab_dofs"] == -(-n_t // gpus) * Ns
