"""bench.py's N>1 orchestration on the one GPU this run has: two ranks under torchrun share cuda:0 with the
gloo backend (collectives bounce through host memory). Checks the partition -> per-rank kernels -> exchange
-> max-over-ranks timing -> one JSON line on rank 0 path end to end; the numbers are not a
performance measurement."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,overlap,banked", [("flickr", True, "1"), ("tiny", True, "1"), ("flickr", False, "1"),
                                                   ("flickr", True, "2"), ("flickr", False, "2")])
def test_bench_two_ranks_gloo(config, overlap, banked, tmp_path):
    """... and the outputs of each rank's last timed step (--dump) against the fp64 oracle: the rank's CBSR block
    bit-exact, its rows of Y and dXs within the north-star bar (all rows of tiny, sampled rows of Flickr).
    banked = "2": the forward reads the bank-balanced copy on both ranks (forced; k = 32)."""
    port = str(29641 + ["flickr-True-1", "tiny-True-1", "flickr-False-1", "flickr-True-2", "flickr-False-2"].index(
        f"{config}-{overlap}-{banked}"))
    k = 32 if banked == "2" else (16 if config == "flickr" else 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", port,
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
           "--config", config, "--k", str(k), "--dist-backend", "gloo", "--dump", str(tmp_path)]
    if not overlap:
        cmd.append("--no-overlap")
    env = dict(os.environ, MAXK_BANKED=banked)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 3
    assert d["collectives"]["allgather"]["bytes"] > 0 and d["collectives"]["reducescatter"]["bytes"] > 0
    assert d["gpu_launches"] > 0 and "dist_backend" in d["config"]
    assert ("overlap" in d) == overlap  # f2 local/remote split is the default for N > 1

    # parity of the timed run, per rank (outputs dumped after the timed region)
    cfg = synth.CONFIGS[config]
    g = synth.config_graph(config)
    x = synth.normal_f32((cfg.n, cfg.h), synth.X_SEED)
    dy = synth.normal_f32((cfg.n, cfg.h), synth.DY_SEED)
    rd, ri = oracle.topk_cbsr(x, k)
    for rank in range(2):
        z = np.load(tmp_path / f"rank{rank}.npz")
        r0, r1 = int(z["r0"]), int(z["r1"])
        assert bool(z["banked"]) == (banked == "2")
        assert np.array_equal(z["sp_idx"].astype(np.int64), ri[r0:r1])
        assert np.array_equal(z["sp_data"].view(np.uint32), rd[r0:r1].view(np.uint32))
        rows = np.arange(r0, r1) if cfg.n <= 5000 else np.unique(np.linspace(r0, r1 - 1, 400).astype(np.int64))
        for name, got, ref in (("Y", z["y"][rows - r0], oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, cfg.h,
                                                                            rows=rows)),
                               ("dXs", z["dxs"][rows - r0], oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri,
                                                                              rows=rows))):
            err = np.abs(got.astype(np.float64) - ref).max(axis=1)
            tol = 1e-5 * (1.0 + np.abs(ref).max(axis=1))
            assert np.all(err <= tol), f"rank {rank} {name}: worst {float((err / tol).max()):.2f} x tol"
