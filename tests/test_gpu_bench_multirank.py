"""The N>1 path of bench.py (north_star: output-feature shards, no collective
on the GEMM) run under torchrun on a one-GPU box: SLSP_BENCH_SHARE_GPU=1 puts
every rank on cuda:0 and uses gloo for the host collectives (the driver's
scaling run uses NCCL, one GPU per rank). Timings are meaningless here; the
test checks that both the replicated-X and the --sharded-lift variants run to
completion, that rank 0 prints one JSON line with the multi-GPU fields and that
the sharded GEMM outputs pass the bench's own CPU-reference parity check."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("extra", [[], ["--sharded-lift"]])
def test_bench_two_ranks_one_gpu(extra):
    env = dict(os.environ, SLSP_BENCH_SHARE_GPU="1", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu", "--no-dense",
           "--tokens", "1024", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["parity"]["bit_exact"] is True
    assert d["config"]["parallelism"] == "N-shard x2"
