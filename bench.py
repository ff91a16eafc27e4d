#!/usr/bin/env python
"""Benchmark of the MaxK-GNN layer hot path (BASELINE.json metric: ms per MaxK layer, fwd+bwd).

One STEP = one pass of the whole hot path over the synthetic graph:
    top-k -> CBSR of X (Eq. 1) ; [N>1: NCCL all-gather of CBSR] ; SpGEMM fwd Y = A·CBSR (Eq. 3 left) ;
    SSpMM bwd dXs = (A^T dY) at the mask (Eq. 3 right) ; [N>1: NCCL reduce-scatter of dXs partials]
Default workload: the Reddit-shaped graph (N=232,965, nnz~114.6M, H=256, k=32) — BASELINE.json's
metric config. value = device time per layer (max over ranks), inputs resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config reddit] [--k 32] [--impl maxk|reference]

Prints ONE JSON line on rank 0. --impl reference times the CPU oracle (oracle/, fp64) on a bounded
row sample of the same workload, extrapolated to ms per layer (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "ms per MaxK layer (fwd+bwd) and HBM GB/s vs roofline, Reddit-shaped, H=256 k=32"
L2_BYTES = 126 * 1024 * 1024


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--config", default="reddit", choices=sorted(synth.CONFIGS))
    p.add_argument("--k", type=int, default=32)
    p.add_argument("--impl", default="maxk", choices=["maxk", "reference"])
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget-s", type=float, default=15.0)
    p.add_argument("--no-plan", action="store_true")
    p.add_argument("--dump", default=None,
                   help="directory: each rank saves the outputs of its last timed step (its rows of Y and dXs, its "
                        "CBSR block) as rank<r>.npz, for tests/test_gpu_bench_multirank.py's parity check")
    p.add_argument("--no-overlap", action="store_true",
                   help="N>1: run the collectives without the f2 local/remote comm-compute overlap")
    p.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                   help="N > 1: NCCL collectives (default), or p2p: the exchanges fused into the top-k and backward "
                        "kernels over torch symmetric memory (dist.PeerMemoryMaxk; needs an NVLink node)")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="gloo: multi-rank orchestration test on one GPU (collectives bounce through the host)")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_model() -> str:
    """Host CPU model, logical cores and sockets."""
    try:
        txt = open("/proc/cpuinfo").read()
        model = next(l.split(":", 1)[1].strip() for l in txt.splitlines() if l.startswith("model name"))
        sockets = len({l.split(":", 1)[1].strip() for l in txt.splitlines() if l.startswith("physical id")}) or 1
        return f"{model}; {os.cpu_count()} logical cores; {sockets} socket(s)"
    except Exception:
        return f"unknown; {os.cpu_count()} logical cores"


def workload_name(cfg, k, n_gpus):
    return (f"{cfg.name}-shaped synthetic Chung-Lu (gamma={cfg.gamma}) N={cfg.n} nnz~{cfg.nnz} H={cfg.h} k={k} "
            f"idx={'uint8' if cfg.h <= 256 else 'uint16'} val=1/deg X,dY~N(0,1)")


# ------------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self, which):
        setattr(self, which, time.time())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [s for t, s in self.samples if self.t0 is None or (self.t0 - 0.05 <= t <= self.t1 + 0.1)]
        if not rows:
            rows = [s for _, s in self.samples[-3:]]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference): bounded row sample, extrapolated to ms/layer
# ------------------------------------------------------------------------------------------------
class OracleSampler:
    """Times the oracle (as it stands) on S sampled rows per stage; value = ms per full layer."""

    def __init__(self, cfg, k, g, x, dy):
        import oracle  # test infrastructure: only this leg of bench.py may use it
        self.oracle = oracle
        self.cfg, self.k, self.g, self.x, self.dy = cfg, k, g, x, dy
        t = time.perf_counter()
        # whole-graph prerequisites of a sampled step (the CBSR of every neighbour, A^T's CSR)
        self.data, self.idx = oracle.topk_cbsr(x, k)
        self.dense = oracle.densify(self.data, self.idx, cfg.h)
        self.transposed = oracle.transpose(g.row_ptr, g.col_idx, g.val, cfg.n)
        self.setup_s = time.perf_counter() - t
        self.rng = np.random.default_rng(1234)

    def step(self, s_rows: int):
        o, n = self.oracle, self.cfg.n
        rows = np.sort(self.rng.choice(n, size=min(s_rows, n), replace=False)).astype(np.int64)
        t0 = time.perf_counter()
        o.topk_cbsr(self.x[rows], self.k)
        t1 = time.perf_counter()
        y = o.spmm(self.g.row_ptr, self.g.col_idx, self.g.val, self.dense, rows=rows)
        t2 = time.perf_counter()
        dxs = o.sspmm_bwd(self.g.row_ptr, self.g.col_idx, self.g.val, self.dy, self.idx, rows=rows,
                          transposed=self.transposed)
        t3 = time.perf_counter()
        scale = n / rows.size
        self.last = (rows, y, dxs)  # kept for the parity check of the timed GPU run
        return {"ms": (t3 - t0) * scale * 1e3, "topk_ms": (t1 - t0) * scale * 1e3,
                "fwd_ms": (t2 - t1) * scale * 1e3, "bwd_ms": (t3 - t2) * scale * 1e3, "rows": int(rows.size),
                "wall_s": t3 - t0}

    def parity(self, sp_data, sp_idx, y, dxs, tol=1e-5):
        """Parity of the TIMED GPU run (its outputs copied to the host after the timed loop) against this leg's
        oracle results: CBSR idx/data bit-exact on every row (the whole-graph oracle top-k is a prerequisite of the
        sample anyway), Y and dXs on the sampled rows of the last step, bar max_c|gpu-ref| <= tol*(1+max_c|ref|)
        (BASELINE.json north_star; Eq. 3)."""
        rows, y_ref, d_ref = self.last

        def worst(gpu, ref):
            err = np.abs(gpu.astype(np.float64) - ref).max(axis=1)
            return float((err / (tol * (1.0 + np.abs(ref).max(axis=1)))).max()) if ref.size else 0.0

        w_y, w_d = worst(y[rows], y_ref), worst(dxs[rows], d_ref)
        return {"idx_bitexact": bool(np.array_equal(sp_idx.astype(np.int32), self.idx.astype(np.int32))),
                "data_bitexact": bool(np.array_equal(sp_data.view(np.uint32), self.data.view(np.uint32))),
                "cbsr_rows_checked": int(self.cfg.n), "y_rows_checked": int(rows.size),
                "dxs_rows_checked": int(rows.size), "worst_err_over_tol": {"y": w_y, "dxs": w_d},
                "pass": bool(max(w_y, w_d) <= 1.0), "tol": f"{tol}*(1+max|ref|) per row, ref fp64",
                "source": "outputs of the last timed step, copied to the host after the timed region"}

    def calibrate(self, budget_s: float) -> int:
        """Rows per step so one step costs ~budget_s of CPU time (all rows, i.e. a full timed layer, when it fits)."""
        probe = self.step(min(2048, self.cfg.n))
        per_row = probe["wall_s"] / probe["rows"]
        return int(max(256, min(self.cfg.n, budget_s / max(per_row, 1e-9))))

    def sample_desc(self, s_rows):
        if s_rows >= self.cfg.n:
            return (f"the full {self.cfg.name}-shaped layer (all {self.cfg.n} rows per stage: top-k, forward, "
                    f"backward), fp64, timed (not extrapolated); whole-graph CBSR/densify/transpose prerequisites "
                    f"built once ({self.setup_s:.1f}s, not counted)")
        return (f"EXTRAPOLATED: {s_rows} uniformly sampled rows per stage (top-k rows, forward output rows, backward "
                f"CBSR rows) of the {self.cfg.name}-shaped graph, fp64, time x N/{s_rows}; whole-graph "
                f"CBSR/densify/transpose prerequisites built once ({self.setup_s:.1f}s, not counted)")


def load_inputs(cfg, rows=None):
    g = synth.config_graph(cfg.name, rows=rows)
    r0 = 0 if rows is None else rows[0]
    n_local = g.n_rows
    x = synth.normal_f32((n_local, cfg.h), synth.X_SEED, row_offset=r0)
    dy = synth.normal_f32((n_local, cfg.h), synth.DY_SEED, row_offset=r0)
    return g, x, dy


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    import oracle
    g, x, dy = load_inputs(cfg)
    smp = OracleSampler(cfg, args.k, g, x, dy)
    # per-step budget so the whole run ends within ~4 minutes; a full (timed, not extrapolated) layer when it fits
    budget = min(max(args.cpu_budget_s, 12.0), 240.0 / max(1, args.steps + args.warmup))
    s_rows = smp.calibrate(budget)
    for _ in range(args.warmup):
        smp.step(s_rows)
    res = [smp.step(s_rows) for _ in range(args.steps)]
    ms = float(np.mean([r["ms"] for r in res]))
    cores = oracle.num_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.k, world), "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "oracle",
                         "sample": smp.sample_desc(s_rows), "cpu": cpu_model()},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "stages_ms": {k: float(np.mean([r[k] for r in res])) for k in ("topk_ms", "fwd_ms", "bwd_ms")},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# GPU leg
# ------------------------------------------------------------------------------------------------
def traffic_from_profiles(cfg, k, kernel):
    """ncu dram bytes per launch for the dominant kernel, if a committed capture matches this workload."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        return t.get(f"{cfg.name}:k{k}:{kernel}")
    except Exception:
        return None


def counters_from_profiles(cfg, k, stage):
    """Per-launch ncu counters of this build's kernel for (config, k, stage), committed by tools/ncu_counters.py."""
    p = os.path.join(ROOT, "profiles", "ncu_counters.json")
    try:
        with open(p) as f:
            return json.load(f).get(f"{cfg.name}:k{k}:{stage}")
    except Exception:
        return None


def ceilings_from_profiles(cfg, k, fwd_ms, bwd_ms):
    """True-limiter ceilings (tools/ubench.py, committed under profiles/) for this workload, if measured:
    the forward against its shared-memory scatter, the backward against its L2 reductions."""
    p = os.path.join(ROOT, "profiles", "r01", f"ubench_{cfg.name}_k{k}.json")
    try:
        with open(p) as f:
            u = json.load(f)
    except Exception:
        return None
    return {
        "source": os.path.relpath(p, ROOT),
        # the r01 forward ceiling (one per-sub-warp buffer, column-ordered CBSR) bounds that layout only;
        # the replicated buffers over the bank-balanced copy run below it, so only the L1tex fraction applies
        "fwd": {"bound": "l1tex data pipe (see roofline)", "ceiling_ms": None,
                "r01_single_buffer_rmw_ms": u["smem_rmw_ms"]},
        "bwd": {"bound": "L2 reduction throughput (red.global.add.v4, 128 B per edge)", "ceiling_ms": u["red_ms"],
                "frac": u["red_ms"] / bwd_ms},
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2312_08656_b200 import maxk, traffic
    from paper_2312_08656_b200.dist import CudaOps, DistributedMaxk, all_gather_into, max_over_ranks, \
        reduce_scatter_into
    from paper_2312_08656_b200.partition import partition_rows_by_nnz, remap_columns, split_local_remote

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product has no CPU path)")
    gpu = local_rank % torch.cuda.device_count() if args.dist_backend == "gloo" else local_rank
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    maxk.load()
    k, h = args.k, cfg.h

    # ---- inputs: this rank's row block of the graph, X and dY (seeded, synthetic) ----
    t_setup = time.perf_counter()
    deg, _ = synth.power_law_degrees(cfg.n, cfg.nnz, cfg.seed)
    row_ptr_full = np.zeros(cfg.n + 1, np.int64)
    np.cumsum(deg, out=row_ptr_full[1:])
    part = partition_rows_by_nnz(row_ptr_full, world)
    r0, r1 = part.rows(rank)
    g, x_np, dy_np = load_inputs(cfg, rows=(r0, r1) if world > 1 else None)
    col = remap_columns(g.col_idx, part) if world > 1 else g.col_idx
    nnz_local = g.nnz
    rp_d = torch.from_numpy(g.row_ptr).to(dev)
    ci_d = torch.from_numpy(col).to(dev)
    va_d = torch.from_numpy(g.val).to(dev)
    x_d = torch.from_numpy(x_np).to(dev)
    dy_d = torch.from_numpy(dy_np).to(dev)
    ops = CudaOps(rp_d, ci_d, va_d, part.n_slots, h, k, use_plan=not args.no_plan)
    split_ops = None
    if world > 1 and not args.no_overlap:  # f2: local-column edges overlap the all-gather / reduce-scatter
        (lr, lc, lv), (rr, rc, rv) = split_local_remote(g.row_ptr, col, g.val, part, rank)
        split_ops = (CudaOps(*(torch.from_numpy(a).to(dev) for a in (lr, lc, lv)), part.r_max, h, k),
                     CudaOps(*(torch.from_numpy(a).to(dev) for a in (rr, rc, rv)), part.n_slots, h, k))
    agg = DistributedMaxk(part, rank, ops, h, k, dev, split_ops=split_ops)
    pm = None
    if world > 1 and args.exchange == "p2p":  # f2: both exchanges fused into the kernels over peer memory
        from paper_2312_08656_b200.dist import PeerMemoryMaxk, SymmetricPeers
        peers = SymmetricPeers(dist.group.WORLD, part.n_slots, part.r_max, k, agg.sp_idx.dtype, dev)
        pm = PeerMemoryMaxk(part, rank, ops, h, k, peers)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    plan_info = ops.plan.info() if ops.plan is not None else None

    stream = torch.cuda.current_stream()

    def step_timed(ev, stages=True):
        # stages=False (the timed loop): events only at the step boundaries, so consecutive kernels stay adjacent in
        # the stream and programmatic dependent launch overlaps each launch with its predecessor's tail
        # (maxk_internal.cuh); the per-stage breakdown comes from a separate loop with every event recorded
        ev[0].record(stream)
        R = part.r_max
        s0 = rank * R
        # the CBSR pair layout (one rank, k in {8, 16}) or the bank-balanced copy (k in {32, 64, 128}) for the forward
        pairs, banked = agg.sp_pairs, agg.sp_banked
        ops.topk(x_d, agg.sp_data[s0:s0 + agg.n_local], agg.sp_idx[s0:s0 + agg.n_local],
                 None if pairs is None else pairs[s0:s0 + agg.n_local],
                 None if banked is None else tuple(b[s0:s0 + agg.n_local] for b in banked))
        if stages:
            ev[1].record(stream)
        if world > 1:  # what DistributedMaxk.forward gathers: the forward's copy (+ the mask when banked)
            for t in ((*banked, agg.sp_idx) if banked is not None else (agg.sp_data, agg.sp_idx)):
                all_gather_into(t, t[agg._blk])
        if stages:
            ev[2].record(stream)
        ops.forward(*(banked if banked is not None else (agg.sp_data, agg.sp_idx)), agg.y, pairs=pairs)
        if stages:
            ev[3].record(stream)
        ops.backward(dy_d, agg.sp_idx, agg.d_partial)
        if stages:
            ev[4].record(stream)
        if world > 1:
            reduce_scatter_into(agg.d_local, agg.d_partial)
        ev[5].record(stream)

    def step_overlap(ev):  # the f2 pass: top-k + all-gather || local fwd, remote fwd; bwd with RS || local bwd
        ev[0].record(stream)
        agg.forward(x_d)
        ev[1].record(stream)
        agg.backward(dy_d)
        ev[2].record(stream)

    def step_p2p(ev, stages=True):  # PeerMemoryMaxk.step with the stage events between its barrier-separated phases
        ev[0].record(stream)
        pm.peers.barrier()
        pm.topk(x_d)
        pm.peers.barrier()
        if stages:
            ev[1].record(stream)
            ev[2].record(stream)  # the all-gather is inside the top-k
        pm.forward()
        pm.peers.barrier()
        if stages:
            ev[3].record(stream)
        pm.backward(dy_d)
        if stages:
            ev[4].record(stream)
        pm.peers.barrier()  # "reducescatter": the wait until every rank's reductions have landed
        ev[5].record(stream)

    if pm is not None:
        step_timed = step_p2p
        split_ops = None
    step = step_overlap if split_ops is not None else (lambda ev: step_timed(ev, stages=False))
    K, W = args.steps, max(3, args.warmup)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(K)]
    warm = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for _ in range(W):
        step(warm)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(gpu)
    clocks.start()
    time.sleep(0.3)
    launches0 = maxk.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.mark("t0")
    t_start.record(stream)
    for i in range(K):
        step(evs[i])
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks.mark("t1")
    if world > 1:
        dist.barrier()
    launches = maxk.launch_count() - launches0
    clk = clocks.stop()
    # outputs of the timed run, for the parity check in the cpu_baseline leg (host copies, outside the timing)
    snap = None
    if world == 1:
        snap = (agg.sp_data[: agg.n_local].cpu().numpy(), agg.sp_idx[: agg.n_local].cpu().numpy(),
                agg.y.cpu().numpy(), agg.d_partial[: agg.n_local].cpu().numpy())
    if args.dump:
        os.makedirs(args.dump, exist_ok=True)
        r0, r1 = part.rows(rank)
        s0 = rank * part.r_max
        d_out = agg.d_partial if world == 1 else (pm.d_local if pm is not None else agg.d_local)
        y_out = pm.y if pm is not None else agg.y
        np.savez(os.path.join(args.dump, f"rank{rank}.npz"), r0=r0, r1=r1, y=y_out[: agg.n_local].cpu().numpy(),
                 dxs=d_out[: agg.n_local].cpu().numpy(),
                 sp_idx=(pm.sp_idx if pm is not None else agg.sp_idx)[s0:s0 + agg.n_local].cpu().numpy(),
                 sp_data=(pm.sp_data if pm is not None else agg.sp_data)[s0:s0 + agg.n_local].cpu().numpy(),
                 banked=agg.sp_banked is not None and pm is None)
    total_ms = t_start.elapsed_time(t_end)
    overlap_ms = None
    if split_ops is not None:
        overlap_ms = {"fwd_incl_topk_allgather": float(np.mean([evs[i][0].elapsed_time(evs[i][1]) for i in range(K)])),
                      "bwd_incl_reducescatter": float(np.mean([evs[i][1].elapsed_time(evs[i][2]) for i in range(K)]))}
    # the per-kernel / per-collective breakdown (roofline, algbw) comes from separate steps with an event between
    # every stage (not overlapped: the f2 split and PDL's launch overlap are off there), after the timed region
    KB = min(K, 20)
    stage_evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(KB)]
    for i in range(KB):
        step_timed(stage_evs[i])
    torch.cuda.synchronize()
    stage = {name: [e[a].elapsed_time(e[b]) for e in stage_evs]
             for name, a, b in (("topk", 0, 1), ("allgather", 1, 2), ("fwd", 2, 3), ("bwd", 3, 4),
                                ("reducescatter", 4, 5))}
    ms_step = total_ms / K
    if world > 1:
        ms_step = max_over_ranks(ms_step, dev)
    # per-step spread: each step bracketed by its own events on the same stream
    last = 5 if split_ops is None else 2
    per_step = np.array([evs[i][0].elapsed_time(evs[i][last]) for i in range(K)])
    spread = {"median": float(np.median(per_step)), "p10": float(np.percentile(per_step, 10)),
              "p90": float(np.percentile(per_step, 90))}

    # cold-L2 variant (d.7): a 512 MB scrub between steps (not timed), each step timed alone
    cold = None
    if world == 1:
        scrub = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        cold_ms = []
        for _ in range(min(K, 20)):
            scrub.fill_(1.0)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            step_timed(warm)
            c1.record(stream)
            torch.cuda.synchronize()
            cold_ms.append(c0.elapsed_time(c1))
        cold = {"median_ms": float(np.median(cold_ms)), "steps": len(cold_ms), "scrub_bytes": scrub.numel() * 4}
        del scrub

    # ---- e2e: through the public API (HostPipeline) with pinned HOST buffers: every step uploads its X and dY
    # and downloads its Y and dXs inside the timed region; copies overlap compute and each other ----
    from paper_2312_08656_b200.dist import HostPipeline
    x_h = torch.from_numpy(x_np).pin_memory()
    dy_h = torch.from_numpy(dy_np).pin_memory()
    y_h = torch.empty(agg.y.shape, dtype=torch.float32).pin_memory()
    d_h = torch.empty((agg.n_local, k), dtype=torch.float32).pin_memory()
    pipe = HostPipeline(agg)
    for _ in range(2):
        pipe.submit(x_h, dy_h, y_h, d_h)
    pipe.flush()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    pipe.begin()
    KE = max(1, args.e2e_steps)
    for _ in range(KE):
        pipe.submit(x_h, dy_h, y_h, d_h)
    pipe.flush()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / KE
    if world > 1:
        e2e_ms = max_over_ranks(e2e_ms, dev)
    h2d = x_h.numel() * 4 + dy_h.numel() * 4

    # ---- extras (not part of the step): f1 MaxK backward scatter of dXs to a dense N x H gradient ----
    extras = {}
    dx_dense = torch.empty((agg.n_local, h), dtype=torch.float32, device=dev)
    d_src = agg.d_partial[: agg.n_local] if world == 1 else agg.d_local[: agg.n_local]
    s0 = rank * part.r_max
    for _ in range(3):
        maxk.maxk_cbsr_scatter(d_src, agg.sp_idx[s0:s0 + agg.n_local], h, dx=dx_dense)
    xs0 = torch.cuda.Event(enable_timing=True)
    xs1 = torch.cuda.Event(enable_timing=True)
    xs0.record(stream)
    for _ in range(10):
        maxk.maxk_cbsr_scatter(d_src, agg.sp_idx[s0:s0 + agg.n_local], h, dx=dx_dense)
    xs1.record(stream)
    torch.cuda.synchronize()
    t_sc = xs0.elapsed_time(xs1) / 10
    sc_bytes = agg.n_local * (4 * h + (4 + (1 if h <= 256 else 2)) * k)
    extras["cbsr_scatter"] = {"ms": t_sc, "GBps": sc_bytes / (t_sc * 1e-3) / 1e9, "bytes": sc_bytes}
    del dx_dense

    # ---- extras: f4, Eq. 1 fused on tcgen05 (X·W + b -> max-k -> CBSR) vs cuBLAS GEMM + top-k ----
    if h in (128, 256) and k <= 64:
        f_in = 256
        xg = torch.randn((agg.n_local, f_in), device=dev).to(torch.bfloat16)
        wt = (torch.randn((h, f_in), device=dev) / 16).to(torch.bfloat16)
        bias = torch.randn((h,), device=dev)
        sd_f = torch.empty((agg.n_local, k), dtype=torch.float32, device=dev)
        si_f = torch.empty((agg.n_local, k), dtype=agg.sp_idx.dtype, device=dev)
        z_tmp = torch.empty((agg.n_local, h), dtype=torch.float32, device=dev)

        def fused():
            maxk.maxk_linear_topk_cbsr(xg, wt, k, bias=bias, sp_data=sd_f, sp_idx=si_f)

        def unfused():  # one cuBLAS GEMM (bf16 in, fp32 out, bias fused) + the standalone top-k kernel
            z = torch.addmm(bias, xg, wt.t(), out_dtype=torch.float32)
            maxk.maxk_topk_cbsr(z, k, sd_f, si_f)

        def unfused_safe():  # older torch without out_dtype: bf16 GEMM, cast, bias add, top-k
            z = (xg @ wt.t()).float() + bias
            maxk.maxk_topk_cbsr(z, k, sd_f, si_f)

        def t_of(fn, reps=20):
            for _ in range(3):
                fn()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(reps):
                fn()
            a1.record(stream)
            torch.cuda.synchronize()
            return a0.elapsed_time(a1) / reps

        try:
            t_un, base = t_of(unfused), "cuBLAS addmm(bf16->fp32) + maxk_topk_cbsr"
        except Exception:
            t_un, base = t_of(unfused_safe), "torch bf16 mm + cast + bias + maxk_topk_cbsr"
        t_fu = t_of(fused)
        lt_bytes = agg.n_local * f_in * 2 + h * f_in * 2 + agg.n_local * k * (4 + (1 if h <= 256 else 2))
        lt_flops = 2.0 * agg.n_local * f_in * h
        extras["linear_topk_fused"] = {"ms": t_fu, "unfused_ms": t_un, "unfused": base, "speedup": t_un / t_fu,
                                       "GBps": lt_bytes / (t_fu * 1e-3) / 1e9,
                                       "TFLOPs": lt_flops / (t_fu * 1e-3) / 1e12, "f_in": f_in}
        del xg, z_tmp

    # ---- extras: the same pass replayed as a CUDA graph (launch overhead removed; matters for small graphs) ----
    if world == 1:
        from paper_2312_08656_b200.layer import MaxkAggregation
        gagg = MaxkAggregation(rp_d, ci_d, va_d, part.n_slots, h, k)
        graph = gagg.capture_step(x_d, dy_d)
        for _ in range(3):
            graph.replay()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(20):
            graph.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        extras["cuda_graph"] = {"ms": g0.elapsed_time(g1) / 20, "eager_ms": ms_step,
                                "api": "MaxkAggregation.capture_step"}
        del graph
        gagg.close()

    # ---- extras: f4, synthetic 2-layer MaxK-SAGE forward+backward (timing only; random weights/features) ----
    if world == 1 and h in (128, 256) and k <= 64:
        from paper_2312_08656_b200.nn import Graph, MaxKGraphConv
        graph = Graph(rp_d, ci_d, va_d, part.n_slots, h, k)
        feats = torch.randn((agg.n_local, 256), device=dev)
        for fused in (False, True):
            layers = [MaxKGraphConv(256, h, k, fused=fused, device=dev), MaxKGraphConv(h, h, k, fused=fused, device=dev)]

            def model_step():
                out = feats
                for lyr in layers:
                    out = lyr(out, graph)
                out.sum().backward()

            for _ in range(3):
                model_step()
            m0 = torch.cuda.Event(enable_timing=True)
            m1 = torch.cuda.Event(enable_timing=True)
            m0.record(stream)
            for _ in range(5):
                model_step()
            m1.record(stream)
            torch.cuda.synchronize()
            extras["sage2_fwd_bwd_fused" if fused else "sage2_fwd_bwd"] = {
                "ms": m0.elapsed_time(m1) / 5, "layers": 2, "f_in": 256, "h": h, "k": k,
                "gemm": "fused tcgen05 GEMM+top-k fwd, cuBLAS bf16 bwd" if fused else "cuBLAS fp32"}
        del feats, layers
    d2h = y_h.numel() * 4 + d_h.numel() * 4

    # ---- roofline of the dominant kernel (per-launch algorithmic bytes / mean launch time) ----
    peak, peak_src = peaks()
    b = 1 if h <= 256 else 2
    balg = traffic.b_alg(agg.n_local, part.n_slots, nnz_local, h, k, b)
    balg["topk"] = 4 * agg.n_local * h + (4 + b) * agg.n_local * k
    if agg.sp_banked is not None:  # the bank-balanced copy for the forward: k more entries written per row
        balg["topk"] += (4 + b) * agg.n_local * k
    bmin = traffic.b_min(agg.n_local, part.n_slots, nnz_local, h, k, b)
    mean = {kk: float(np.mean(v)) for kk, v in stage.items()}
    # NVLink collectives (N>1): algbw = bytes of the full output / time; busbw = algbw * (N-1)/N (NCCL convention)
    comm = None
    if world > 1:
        ag_bytes = part.n_slots * k * (4 + b + (b if agg.sp_banked is not None else 0))  # + the mask when banked
        rs_bytes = part.n_slots * k * 4
        comm = {}
        for name, nbytes in (("allgather", ag_bytes), ("reducescatter", rs_bytes)):
            t = mean[name] * 1e-3
            alg = nbytes / t / 1e9 if t > 0 else None
            comm[name] = {"ms": mean[name], "bytes": nbytes, "algbw_GBps": alg,
                          "busbw_GBps": alg * (world - 1) / world if alg else None,
                          "busbw_frac_of_900": (alg * (world - 1) / world / 900.0) if alg else None}
    dom = "fwd" if mean["fwd"] >= mean["bwd"] else "bwd"
    vec = k in (8, 16, 32, 64, 96, 128, 192, 256) and os.environ.get("MAXK_FORCE_GENERIC") != "1"
    kernel_name = {"fwd": "spgemm_fwd_kernel" if vec else "spgemm_fwd_generic_kernel",
                   "bwd": "sspmm_bwd_vec_kernel" if vec else "sspmm_bwd_generic_kernel"}[dom]
    achieved = balg[dom] / (mean[dom] * 1e-3) / 1e9
    # per-kernel roofline: the algorithmic-bytes HBM basis (north star), the strict unique-byte
    # basis, DRAM actually moved (ncu), and the resource that binds each kernel -- L1tex data-pipe wavefronts
    # (1 per clock per SM) for the aggregation kernels, warp-instruction issue (4 per clock per SM) for top-k --
    # from the committed ncu counters of this build divided by the LIVE launch time of this run
    sm_hz = (clk or {}).get("sm_mhz", 1965.0) * 1e6 if clk else 1965.0e6
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    kernels = {}
    for st in ("topk", "fwd", "bwd"):
        t = mean[st] * 1e-3
        if t <= 0:
            continue
        c = counters_from_profiles(cfg, k, st) if world == 1 else None
        rec = {"ms": mean[st], "bytes_alg": balg[st], "frac_alg_hbm": balg[st] / t / 1e9 / peak,
               "bytes_min": bmin.get(st), "frac_min_hbm": (bmin[st] / t / 1e9 / peak) if st in bmin else None}
        if c:
            rec["counters"] = c.get("source")
            rec["dram_GBps"] = c["dram_bytes"] / t / 1e9
            rec["frac_dram"] = rec["dram_GBps"] / peak
            if c.get("l1tex_wavefronts"):
                rec["l1tex_wavefronts"] = c["l1tex_wavefronts"]
                rec["frac_l1tex"] = c["l1tex_wavefronts"] / t / (n_sm * sm_hz)
            if c.get("smem_wavefronts"):
                rec["smem_wavefronts_per_edge"] = c["smem_wavefronts"] / max(1, nnz_local)
            if c.get("inst"):
                rec["frac_issue"] = c["inst"] / t / (4 * n_sm * sm_hz)
            if c.get("lts_red_sectors"):
                rec["l2_red_GBps"] = c["lts_red_sectors"] * 32 / t / 1e9
            cands = {kk: rec[v] for kk, v in (("l1tex", "frac_l1tex"), ("issue", "frac_issue"), ("hbm", "frac_dram"))
                     if v in rec}
            rec["binding"] = max(cands, key=cands.get) if cands else None
        kernels[st] = rec
    trf = traffic_from_profiles(cfg, k, kernel_name)
    dc = counters_from_profiles(cfg, k, dom) if world == 1 else None
    if dc:
        trf = dc["dram_bytes"]
    kd = kernels.get(dom, {})

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    layer_balg = traffic.b_alg(cfg.n, cfg.n, cfg.nnz, h, k, b)["layer"]
    layer_bmin = traffic.b_min(cfg.n, cfg.n, cfg.nnz, h, k, b)["layer"]
    line = {
        "metric": METRIC,
        "value": ms_step,
        "unit": "ms",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": ms_step,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {
            "workload": workload_name(cfg, k, world),
            "nnz": int(row_ptr_full[-1]),
            "parallelism": (f"rows{world} (nnz-balanced row blocks; CBSR all-gather fused into the top-k and dXs "
                            "reduce-scatter fused into the backward, over symmetric memory)" if pm is not None else
                            f"rows{world} (nnz-balanced row blocks; NCCL all-gather CBSR + reduce-scatter dXs)")
            if world > 1 else "1 GPU",
            "l2": "inputs larger than L2 (X, dY, CSR = %.2f GB > 126 MB); no flush" % (
                (x_np.nbytes + dy_np.nbytes + g.row_ptr.nbytes + col.nbytes + g.val.nbytes) / 1e9),
            "plan": plan_info,
            **({"dist_backend": "gloo (host-bounced collectives, ranks may share a GPU): orchestration test, "
                                "not a performance number"} if world > 1 and args.dist_backend == "gloo" else {}),
        },
        "roofline": ({
            # the resource that binds the dominant kernel: L1tex data-pipe wavefronts of this
            # build (committed ncu capture, profiles/ncu_counters.json) per LIVE launch time, against
            # 1 wavefront / clock / SM x SMs at the clock sampled during the timed region
            "bound": "l1tex",
            "kernel": kernel_name,
            "achieved": kd["l1tex_wavefronts"] / (mean[dom] * 1e-3) / 1e9,
            "peak": n_sm * sm_hz / 1e9,
            "unit": "Gwavefronts/s",
            "frac": kd["frac_l1tex"],
            "traffic": trf,
            "hbm_basis": {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac_alg": achieved / peak,
                          "frac_min": kd.get("frac_min_hbm"), "dram_GBps": kd.get("dram_GBps"),
                          "bytes_alg_per_launch": balg[dom], "peak_source": peak_src,
                          "note": "algorithmic bytes (SURVEY §8(d) d.5, the north-star basis) count every CBSR "
                                  "gather; most hit in L2, so this is not DRAM traffic"},
        } if kd.get("frac_l1tex") is not None else {
            "bound": "hbm",
            "kernel": kernel_name,
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": trf,
            "bytes_alg_per_launch": balg[dom],
            "peak_source": peak_src,
            "note": "no committed ncu counters for this workload: algorithmic-bytes basis only",
        }),
        "kernels": kernels,
        "layer_roofline": {
            "bytes_alg": layer_balg, "frac_alg": layer_balg / (ms_step * 1e-3) / 1e9 / peak,
            "bytes_min": layer_bmin, "frac_min": layer_bmin / (ms_step * 1e-3) / 1e9 / peak,
        },
        "step_ms_spread": spread,
        "cold_l2": cold,
        "stages_ms": mean,
        **({"overlap": {"mode": "f2: local-column edges during the all-gather, local-target edges during the "
                                "reduce-scatter; stages_ms from separate non-overlapped steps", "ms": overlap_ms}}
           if overlap_ms is not None else {}),
        "collectives": comm,
        "ceilings": ceilings_from_profiles(cfg, k, mean["fwd"], mean["bwd"]),
        "edges_k_per_s": cfg.nnz * k / (ms_step * 1e-3),
        "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": KE, "api": "paper_2312_08656_b200.dist.HostPipeline (copies overlapped across steps)"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "setup_s": setup_s,
        "extras": extras,
        "context": {"paper_a100_ms_per_layer_real_reddit": 30.82,
                    "note": "PAPER.md:686 Table 5 (A100, real Reddit): MaxK 0.261 + SpGEMM 15.49 + SSpMM 15.07 ms"},
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            smp = OracleSampler(cfg, k, g, x_np, dy_np)
            s_rows = smp.calibrate(args.cpu_budget_s)
            r = smp.step(s_rows)
            runs = [r["ms"]]
            if r["wall_s"] * 2 <= args.cpu_budget_s:  # median of 3 when affordable
                runs += [smp.step(s_rows)["ms"] for _ in range(2)]
            line["cpu_baseline"] = {"value": float(np.median(runs)), "unit": "ms", "cores": oracle.num_threads(),
                                    "kind": "oracle", "runs": len(runs), "sample": smp.sample_desc(s_rows),
                                    "cpu": cpu_model()}
            if cfg.n <= 100_000:  # tiny / Flickr-shaped: also the single-thread oracle (d.8)
                nt = oracle.num_threads()
                oracle.set_num_threads(1)
                line["cpu_baseline"]["one_thread_ms"] = smp.step(cfg.n)["ms"]
                oracle.set_num_threads(nt)
            if snap is not None:
                line["parity"] = smp.parity(*snap)
        except Exception as e:  # the baseline is reported context; never let it kill the bench line
            line["cpu_baseline"] = {"value": None, "unit": "ms", "cores": None, "kind": "oracle",
                                    "sample": f"failed: {e}"}
    print(json.dumps(line), flush=True)
    ops.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
