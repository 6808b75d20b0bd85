"""bench.py's data-parallel harness with world size 2: two ranks on the one GPU of the
test box over gloo (NCCL needs a GPU per rank), real encoder kernels, the max-over-ranks timing and the
score gather -- the code path `torchrun --nproc-per-node N bench.py` takes on an 8-GPU node."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_world2_gloo_one_gpu():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--steps", "2", "--warmup", "3", "--pairs-per-gpu", "2",
           "--no-variants", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 4 and d["config"]["parallelism"] == "dp2"
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    # rank 0's own scores (pairs 0, 1 of the reference golden) through the gathered step
    assert d["parity"]["n"] == 2 and d["parity"]["max_abs_err"] < 2e-2
