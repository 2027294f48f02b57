"""Device multi-rank H_eff·ψ (sharded plans + all-reduce) under torchrun.
On a 1-GPU box the ranks share cuda:0 over gloo; with >= 2 GPUs the same
check runs over NCCL, one rank per GPU."""

import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_apply_allreduce_equals_full(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ)
    if torch.cuda.device_count() < world:
        env["SDMRG_DIST_BACKEND"] = "gloo"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(_port()), os.path.join(ROOT, "tools", "check_multirank.py"),
           "12", "64"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "PASS" in out.stdout


def test_bench_two_ranks_sector_shards():
    """bench.py under torchrun with two ranks (sharing cuda:0 over gloo on a
    1-GPU box): per-rank arenas generated in place, the max-over-ranks
    timing and one JSON line from rank 0."""
    import json
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ)
    if torch.cuda.device_count() < 2:
        env["SDMRG_DIST_BACKEND"] = "gloo"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--L", "16", "--D", "256", "--scale", "", "--sweep", "", "--no-e2e"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["operator_arena_gb_per_rank_max"] > 0
