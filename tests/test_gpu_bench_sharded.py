"""bench.py's sharded path end to end with two ranks (torchrun, one process per rank): item-range
shards, the single-device threshold exchange (each rank's top-n sample keys all-gathered, the
n-th largest of the union), the per-shard two-stage retrieval, the all-gather of (ids, scores)
and molr_merge_top_k.  On a one-GPU box both ranks share cuda:0 and the collectives run over gloo
(MOLR_BENCH_SHARE_GPU=1; NCCL refuses two ranks on one device) — the same device tensors and
calls as the NCCL run.  The merged top-k of the whole batch must be bit-identical to the one-rank
run (result digest over ids and score bits)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(nproc, extra):
    args = ["--config", "10m", "--items", "400000", "--steps", "2", "--warmup", "1", "--no-cpu", "--no-oracle",
            "--recall-queries", "4", "--gpus", str(nproc)] + extra
    env = dict(os.environ, MOLR_BENCH_SHARE_GPU="1")
    if nproc == 1:
        cmd = [sys.executable, "bench.py"] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py"] + args
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_two_rank_bench_equals_one_rank():
    one = _run(1, [])
    two = _run(2, ["--global-threshold"])
    assert two["n_gpus"] == 2 and two["value"] > 0
    assert two["config"]["threshold"].startswith("single-device")
    assert two["result_digest_step0"] == one["result_digest_step0"]
    assert two["recall_at_k_vs_exact_mol"] >= 0.99
