"""bench.py's multi-rank paths, run functionally with two ranks sharing one GPU over gloo (the
driver's N-GPU runs use NCCL, one GPU per rank): batch x head weak (config 2) and strong (config 4)
sharding and the sequence-parallel step (config 3: segment summaries, all-gather, compose, local
scans).  Checks the JSON contract line; the times are meaningless here (two ranks, one GPU)."""
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


@pytest.mark.parametrize("cfg,scaling", [("2", "weak"), ("4", "strong"), ("3", "strong")])
def test_bench_two_ranks_gloo(cfg, scaling):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", cfg,
           "--dist-backend", "gloo", "--steps", "2", "--warmup", "1", "--seeds", "1", "--stat-steps", "2",
           "--no-cpu-baseline", "--no-e2e", "--no-layer", "--profile"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0
    assert d["config"]["config_id"] == int(cfg)
    if cfg == "3":
        assert d["config"]["parallelism"].startswith("sp2")
        assert d["config"]["seq_len_per_gpu"] == 17984 // 2
