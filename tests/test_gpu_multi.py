"""The distributed path on >= 2 GPUs (skipped on a one-GPU box): tools/dist_check.py under
torchrun, the gathered slabs of fd_apply (NCCL and fused all-to-all), ls_matvec and the
PCG iterate against a single-GPU context, cube and mapped domain."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("extra", [[], ["--a2a", "fused"], ["--geometry", "--n-el", "8", "--p", "2"]])
@pytest.mark.parametrize("world", [2, 4])
def test_distributed_matches_single_gpu(world, extra):
    if world > _ngpu():
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "dist_check.py")]
    out = subprocess.run(cmd + extra, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    res = json.loads(line)
    assert res["fd_rel"] <= 1e-12 and res["matvec_rel"] <= 1e-12, res
    assert res["fd_after_matvec_rel"] <= 1e-12, res
    assert all(it == res["iters_1gpu"] for it in res["iters"]), res
    assert res["pcg_rel"] <= 1e-9, res
