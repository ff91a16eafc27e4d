"""bench.py's N>1 orchestration on the one GPU this run has: two ranks under torchrun share cuda:0 with the
gloo backend (collectives bounce through host memory). Checks the partition -> per-rank kernels -> exchange
-> max-over-ranks timing -> one JSON line on rank 0 path end to end; the numbers are not a
performance measurement."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,overlap", [("flickr", True), ("tiny", True), ("flickr", False)])
def test_bench_two_ranks_gloo(config, overlap):
    port = {("flickr", True): "29641", ("tiny", True): "29642", ("flickr", False): "29643"}[(config, overlap)]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", port,
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
           "--config", config, "--k", "16" if config == "flickr" else "8", "--dist-backend", "gloo"]
    if not overlap:
        cmd.append("--no-overlap")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 3
    assert d["collectives"]["allgather"]["bytes"] > 0 and d["collectives"]["reducescatter"]["bytes"] > 0
    assert d["gpu_launches"] > 0 and "dist_backend" in d["config"]
    assert ("overlap" in d) == overlap  # f2 local/remote split is the default for N > 1
