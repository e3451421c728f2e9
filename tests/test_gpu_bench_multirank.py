"""The bench's N > 1 path end to end (torchrun, 2 ranks) on a one-GPU box:
both ranks on cuda:0 with gloo (GES_BENCH_DEVICE / GES_BENCH_BACKEND are
test-only overrides; not a measurement).  Covers the peer-memory frame gather
and the collective fallback to the NCCL/gloo gather when a rank cannot map
the peer buffer (GES_BENCH_PEER_FAIL)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(extra_env, extra_args=()):
    env = dict(os.environ, GES_BENCH_DEVICE="0", GES_BENCH_BACKEND="gloo", **extra_env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--config", "1", "--views", "2", "--streams", "2", "--steps", "2", "--warmup", "3",
           "--no-cpu", "--no-e2e", *extra_args]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]   # rank 0 alone prints
    return json.loads(lines[0]), p.stderr


@pytest.mark.gpu
def test_bench_two_ranks_peer_gather():
    d, _ = _run({})
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["frame_gather"].startswith("peer")


@pytest.mark.gpu
def test_bench_two_ranks_peer_fallback():
    d, err = _run({"GES_BENCH_PEER_FAIL": "1"})
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert "peer buffer unavailable" in d["config"]["frame_gather"]
    assert "using the NCCL gather" in err


@pytest.mark.gpu
@pytest.mark.parametrize("fail", [False, True])
def test_bench_two_ranks_screen_strips(fail):
    """--strips: one frame per step, two row bands, peer gather (or the padded
    NCCL/gloo gather when the peer buffer is unavailable)."""
    d, _ = _run({"GES_BENCH_PEER_FAIL": "1"} if fail else {}, ("--strips",))
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["config"]["parallelism"] == "row strips x2"
    assert [tuple(b) for b in d["config"]["strips"]] == [(0, 64), (64, 128)]
