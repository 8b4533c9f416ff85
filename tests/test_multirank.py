"""The multi-GPU launcher path, executed: bench.py under torchrun with two
ranks on one GPU (BVP_BENCH_BACKEND=gloo -- the same code path as NCCL on an
8-GPU box, minus the transport).  Each rank pools its own sample(s); rank 0
reports the max over ranks, the per-rank device times, and verifies the
gathered maps against single-process recomputation."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(*bench_args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--no-variants", "--no-cpu-baseline",
           *bench_args]
    env = dict(os.environ, BVP_BENCH_BACKEND="gloo")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_two_ranks_config_S():
    line = _torchrun("--steps", "3", "--warmup", "3")
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    mr = line["multi_rank"]
    assert len(mr["per_rank_step_ms"]) == 2 and all(t > 0 for t in mr["per_rank_step_ms"])
    assert mr["gathered_maps_bit_identical_to_single_process"] is True
    assert line["ms_per_step"] >= max(mr["per_rank_step_ms"]) - 1e-9  # max over ranks


@pytest.mark.parametrize("config", ["F", "B", "H"])
def test_two_ranks_configs_F_B_H(config):
    line = _torchrun("--config", config, "--steps", "2", "--warmup", "3")
    assert line["n_gpus"] == 2
    assert len(line["latency_ms"]["per_rank_step_ms"]) == 2
    assert line["config"]["batch_per_gpu"] == (4 if config == "B" else 1)
