"""bench.py's N > 1 path run for real: two ranks (torchrun, gloo with
host-staged messages, both on the one GPU of the box) -- the row-strip
config-4 step and the image-per-GPU config-5 split -- print one well-formed
JSON line from rank 0."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_gloo():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--size", "1024",
           "--dist-backend", "gloo"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["parallelism"] == "row-strips x2"
    c5 = d["config5"]
    assert c5["n_gpus"] == 2 and c5["images_per_gpu"] == 32 and c5["image_iters_per_s"] > 0
    assert set(c5["oracle_images"]) == {"img0"}       # rank 0 holds images 0..31
    assert abs(c5["oracle_images"]["img0"]["psnr_diff_db"]) < 0.02
