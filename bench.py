#!/usr/bin/env python
"""bench.py -- outer-product terms counted per second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

A step is one pass of the hot path over the whole synthetic workload of the
configuration (default c2 = BASELINE.json configs[1], the 1-GPU exact pair
count): per-item term scan + tile plan, routing, shared-memory counting of
every pair term (i < j) of the GPU's tile share, the per-bucket top-l
Space-Saving summaries when the config bounds them (c3: l = 65,536 per
bucket), and the top-k select. `--config c3|c4|c5` measures the other
configurations (c4 through the real-valued product path).
Inputs are resident in HBM; L2 is flushed (1 GiB write) before every timed
step. `value` = all terms of the workload / (max over ranks of the summed
per-step CUDA-event time). `e2e` runs the public API (`crop.run` +
`SketchState.top_entries`) from pinned host buffers, host<->device copies
inside the timed region. `roofline` is the counting path of SURVEY.md §8(d)
(B_alg = 8 B/term + input + output over the path's live CUDA-event time),
with each phase's kernels, time and share of the step. `cpu_baseline` is the
C oracle (the reference algorithm restated, oracle/crop_oracle.c) on a
bounded prefix, shared-nothing threads on the host cores.

Under torchrun (N > 1) rank 0 generates the workload and broadcasts it once
over NCCL; every rank plans the same tiles and counts its 1/N share of them
by terms (no communication; the shards are disjoint and cover the job);
local top-k candidates are all-gathered and merged on rank 0.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "outer-product terms counted/sec at 1/2/4/8 B200; % of HBM roofline"
HBM_FALLBACK_GBS = 6650.0
SUB_SHARD_CAPACITY = 1_500_000_000  # output entries per sub-shard (c3), 18 GB


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--cpu-sample-tx", type=int, default=None,
                    help="transactions in the CPU-baseline sample (default per config)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers

def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region:
    ONE `nvidia-smi -lms` process (the profiling recipe's clocks line), started
    when the sampler is made -- before the warm-up steps -- so that no
    process is spawned inside the timed region (a fork + nvidia-smi start-up
    per sample perturbed the host-side launches of short steps: c4 measured
    2.1 to 3.2 ms with it). `with sampler:` marks the timed window; the
    summary uses the samples inside it (or the nearest ones when the window
    is shorter than the sampling period)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    PERIOD_MS = 100

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []  # (wall time, fields)
        self.t0 = self.t1 = None
        self._proc = None
        self._t = None
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None

    def _read(self):
        try:
            for line in self._proc.stdout:  # blocks in read(): the GIL is released
                parts = [x.strip() for x in line.strip().split(",")]
                if len(parts) >= 9:
                    self.samples.append((time.time(), parts))
        except Exception:
            pass

    def __enter__(self):
        self.t0 = time.time()
        return self

    def __exit__(self, *exc):
        self.t1 = time.time()
        # one more period so a sample taken under the last steps' load arrives
        time.sleep(self.PERIOD_MS / 1000.0)
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            if self._t is not None:
                self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        inside = [f for t, f in self.samples if self.t0 is not None and self.t0 <= t <= self.t1]
        if not inside and self.t0 is not None:
            # window shorter than the period: the samples next to it
            mid = 0.5 * (self.t0 + self.t1)
            inside = [f for _, f in sorted(self.samples, key=lambda tf: abs(tf[0] - mid))[:2]]
        sm = [float(s[1]) for s in inside if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in inside if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in inside for k in range(4) if s[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(inside), "period_ms": self.PERIOD_MS}


def ncu_traffic(config: str):
    """DRAM bytes (read + write) of one counting path from the committed ncu
    summary (profiles/ncu_summary.json, `ncu --set full` per kernel), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d[config]["path_dram_bytes"]
    except Exception:
        return None


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def config_dict(cfg, world):
    """The workload description both arms print (identical dicts)."""
    from paper_1210_0461_b200 import workloads

    if isinstance(cfg, workloads.PairConfig):
        return {"workload": cfg.name, "n_tx": cfg.n_tx, "n_items": cfg.n_items,
                "zipf_s": cfg.zipf_s, "length": list(cfg.length), "kappa": cfg.kappa,
                "top_k": cfg.top_k, "ss_capacity": cfg.ss_capacity, "data_seed": cfg.seed,
                "engine_seed": 0, "upper_triangle_only": True,
                "parallelism": (f"stream-chunks{world}" if cfg.ss_capacity and world == 1
                                else f"tiles{world}"),
                "l2": "flushed (1 GiB write) before every timed step"}
    return {"workload": cfg.name, "n": cfg.n, "kappa": cfg.kappa, "data_seed": cfg.seed,
            "engine_seed": 0, "parallelism": f"buckets{world}",
            "l2": "flushed (1 GiB write) before every timed step"}


# ------------------------------------------------------------------ workload

def load_workload(cfg, rank, world):
    """Device transactions on every rank (rank 0 generates, NCCL broadcast)."""
    import torch

    from paper_1210_0461_b200 import kernels, workloads

    if world == 1:
        return workloads.generate_pairs_workload(cfg), 0.0
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device())
    if rank == 0:
        dtx = workloads.generate_pairs_workload(cfg)
        sizes = torch.tensor([dtx.n_tx, dtx.nnz], dtype=torch.int64, device=dev)
    else:
        sizes = torch.zeros(2, dtype=torch.int64, device=dev)
    dist.broadcast(sizes, 0)
    n_tx, nnz = int(sizes[0]), int(sizes[1])
    if rank != 0:
        dtx = kernels.DeviceTransactions(torch.empty(n_tx + 1, dtype=torch.int64, device=dev),
                                         torch.empty(nnz, dtype=torch.int32, device=dev),
                                         cfg.n_items)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    dist.broadcast(dtx.offsets, 0)
    dist.broadcast(dtx.items, 0)
    torch.cuda.synchronize()
    return dtx, time.perf_counter() - t0


# ------------------------------------------------------------------ our arm

def run_ours(args, rank, world):
    import numpy as np
    import torch

    import paper_1210_0461_b200 as crop
    from paper_1210_0461_b200 import kernels, workloads

    cfg = workloads.CONFIGS[args.config]
    if not isinstance(cfg, workloads.PairConfig):
        return run_product(args, rank, world)
    dev = torch.device("cuda", torch.cuda.current_device())
    dtx, bcast_s = load_workload(cfg, rank, world)
    if cfg.ss_capacity and world == 1:
        return run_streaming_summaries(args, cfg, dtx)
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.workers,
                               cs_enabled=False, seed=0)
    hasher = crop.make_hashes(crop.HashConfig(cfg.kappa, config.instance_seeds()[0]))
    tables = kernels.hash_tables(hasher, cfg.n_items)
    # rank r counts its 1/N share of the planned tiles (all buckets); the
    # shards are disjoint and cover the job (crop_pairs_create_sharded)
    interval = None
    shard = (rank, world)
    flush = torch.empty(1 << 28, dtype=torch.int32, device=dev)  # 1 GiB > 126 MB L2

    def step():
        # counting path (SURVEY.md §8d primary time): from the first kernel of
        # the job (per-item term scan) to the last counting kernel
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        try:
            job = kernels.PairCountJob(dtx, True, interval, keep=tables, shard=shard)
        except crop.ResourceCapError:
            # the shard's entry lists exceed one job's 2^32 limit (c3): count it
            # as consecutive sub-shards (kernels.count_pairs_shard)
            job = None
            ent = kernels.count_pairs_shard(dtx, True, interval, keep=tables, shard=shard,
                                            capacity=SUB_SHARD_CAPACITY)
            p1.record()
        if job is not None:
            job.set_timing(True)
            ent = job.run(sync=False)
            p1.record()

        def settle():
            # the entry count is read back after the top-k launches when the
            # select runs on the device-side count (one synchronisation less)
            if job is not None:
                ent.n = int(ent.n_dev.item())
                if ent.n > ent.capacity or job.overflowed():
                    raise RuntimeError("pair engine overflow")

        src, cnt = ent, None
        if cfg.ss_capacity:
            settle()
            # bounded Space-Saving regime (c3): per-bucket top-l summaries. With
            # N > 1 every bucket's pairs are spread over the tile shards: each
            # rank sends its per-bucket candidates to the bucket's owner (one
            # all-to-all) and the owner selects the bucket's top-l
            if world > 1:
                from paper_1210_0461_b200 import distributed

                cand, mask, _, _, _ = distributed.merge_bucket_summaries_distributed(
                    ent, tables[0], tables[1], cfg.kappa, cfg.ss_capacity)
                src = cand
                cnt = torch.where(mask, cand.count[: cand.n], torch.zeros_like(cand.count[: cand.n]))
            else:
                mask, _, _ = kernels.bucket_topk(ent, tables[0], tables[1], cfg.kappa, cfg.ss_capacity)
                cnt = torch.where(mask, ent.count[: ent.n], torch.zeros_like(ent.count[: ent.n]))
        idx = kernels.topk_indices(src, cfg.top_k, count=cnt)
        if not cfg.ss_capacity:
            settle()
        top = (src.row[idx], src.col[idx], src.count[idx])
        if world > 1:
            import torch.distributed as dist

            # gather every rank's local top-k; rank 0 selects the global top-k
            # (count desc, row, col) with the same device select
            k = cfg.top_k
            buf = torch.full((3, k), -1, dtype=torch.int32, device=dev)
            m = idx.shape[0]
            buf[0, :m], buf[1, :m], buf[2, :m] = top
            allb = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(allb, buf)
            if rank == 0:
                g = torch.cat(allb, dim=1)
                valid = g[2] != -1
                ge = kernels.DeviceEntries(g[0][valid].contiguous(), g[1][valid].contiguous(),
                                           g[2][valid].contiguous(), None, int(valid.sum().item()), 0)
                gi = kernels.topk_indices(ge, k)
                top = (ge.row[gi], ge.col[gi], ge.count[gi])
        if job is None:
            phases = {"path": p0.elapsed_time(p1), "plan": float("nan"), "route": float("nan"),
                      "write": float("nan"), "count": float("nan")}
            stats = (ent.total_terms, ent.n, None, None, False, ent.sub_shards)
            return phases, stats, top
        phases = job.phase_ms()
        phases["path"] = p0.elapsed_time(p1)
        phases["plan"] = phases["path"] - phases["route"] - phases["write"] - phases["count"]
        stats = (job.total_terms, ent.n, job.n_tiles, job.n_units, job.stream_mode, 1)
        job.close()
        return phases, stats, top

    sampler = ClockSampler(torch.cuda.current_device())  # started before the warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    step_ms, count_ms, phase_log = [], [], []
    launches0 = kernels.launch_counter()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        for k in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            ev[k][0].record()
            phases, stats, top = step()
            ev[k][1].record()
            torch.cuda.synchronize()
            step_ms.append(ev[k][0].elapsed_time(ev[k][1]))
            count_ms.append(phases["count"])
            phase_log.append(phases)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = kernels.launch_counter() - launches0
    total_terms_all = int(((dtx.offsets[1:] - dtx.offsets[:-1]) *
                           (dtx.offsets[1:] - dtx.offsets[:-1] - 1) // 2).sum().item())
    t_sum = sum(step_ms)
    own_terms, own_entries = None, stats[1]
    if world > 1:
        t = torch.tensor([t_sum], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_sum = float(t.item())
    ms_per_step = t_sum / args.steps
    value = total_terms_all * args.steps / (t_sum * 1e-3)

    # roofline: B_alg = 8 B per term (one 4-byte counter read
    # + write) + the input read once + 12 B per output (row, col, count) entry,
    # over the counting path's live CUDA-event time (first kernel of the job to
    # the last counting kernel, host planning gap included). Own terms = terms
    # of this rank's buckets = the sum of its output counts.
    if world > 1:
        ent = kernels.count_pairs_shard(dtx, True, interval, keep=tables, shard=shard,
                                        capacity=SUB_SHARD_CAPACITY)
        own_terms = int(ent.weights_f64().sum().item())
        del ent
    else:
        own_terms = total_terms_all
    # per-partition balance (BASELINE c5: max/mean terms per partition), the
    # LoadReport.max_avg_ratio arithmetic (engine.py:207-216) over the kappa
    # bucket loads of this rank's entries (summed over ranks)
    ent_b = kernels.count_pairs_shard(dtx, True, interval, keep=tables, shard=shard,
                                      capacity=SUB_SHARD_CAPACITY)
    bl, _, _ = kernels.entry_bucket_stats(ent_b, [tables], cfg.kappa, cfg.n_items, None)
    bl = bl[0]
    if world > 1:
        dist.all_reduce(bl)
    del ent_b
    bucket_loads = [int(x) for x in bl.cpu().tolist()]
    balance = {"partitions": cfg.kappa,
               "max_mean": crop.LoadReport(kappa=cfg.kappa, workers=cfg.kappa, rows=[bucket_loads],
                                           input_pair_total=0).max_avg_ratio(),
               "max_terms": max(bucket_loads), "mean_terms": sum(bucket_loads) / cfg.kappa,
               "source": "exact bucket loads of the counted entries (sum of supports per "
                         "bucket), LoadReport.max_avg_ratio arithmetic"}
    in_bytes = 4 * int(dtx.items.numel()) + 8 * int(dtx.offsets.numel())
    b_alg = 8 * own_terms + in_bytes + 12 * own_entries
    avg = {k: statistics.mean(p[k] for p in phase_log) for k in phase_log[0]}
    peak, peak_src = peaks()
    achieved = b_alg / (avg["path"] * 1e-3) / 1e9
    stream_mode = bool(stats[4])
    if stats[5] > 1:
        mode_name = f"entry, {stats[5]} sub-shards per GPU"
    else:
        mode_name = "stream" if stream_mode else "entry"
    kern = {"plan": ("k_item_terms + k_plan_coop (device planner) + plan read-back" if stream_mode
                     else "k_item_terms + host tile plan + uploads"),
            "route": "k_scan_u64 (+ k_stream_count when word totals are unknown)" if stream_mode
                     else "k_route",
            "write": "k_chunk_bounds + k_stream_scatter (or k_stream_write)" if stream_mode
                     else "k_tile_entries",
            "count": "k_count_stream + k_reduce_slabs" if stream_mode else "k_count"}
    roofline = {"bound": "hbm", "kernel": "counting path: " + " -> ".join(kern[k] for k in
                                                                          ("plan", "route", "write", "count")),
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.config),
                "peak_source": peak_src, "algorithmic_bytes_per_launch": b_alg,
                "avg_launch_ms": round(avg["path"], 4),
                "phases": {k: {"kernels": kern[k], "ms": round(avg[k], 4),
                               "share_of_step": round(avg[k] / ms_per_step, 4)}
                           for k in ("plan", "route", "write", "count") if avg[k] == avg[k]},
                "mode": mode_name}

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, dtx, rank, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, cfg, dtx)

    if rank == 0:
        line = {
            "metric": BASELINE_METRIC, "value": value, "unit": "terms/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic: seeded Zipf transactions (SURVEY.md §8d, data seed = config no.)",
            "config": config_dict(cfg, world),
            "details": {"sharding": f"tiles split by terms over {world} GPU(s), all {cfg.kappa} buckets",
                        "terms": total_terms_all, "entries": own_entries if world == 1 else None,
                        "tiles": stats[2], "units": stats[3], "broadcast_s": round(bcast_s, 4)},
            "partition_balance": balance,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)


STREAM_CHUNK_TX = 8_333_334  # c3: 6 chunks of ~3.75e9 terms (measured: 10 chunks 1.71 s, 6 chunks 1.50 s, 5 chunks 1.62 s)


def run_streaming_summaries(args, cfg, dtx):
    """c3 on one GPU: the bounded Space-Saving regime with O(l) summary
    state (kernels.StreamingSummaries, the loop of crop.run_streaming). A
    step counts every chunk of transactions exactly on chip and merges it
    into the kappa per-bucket summaries of l records, then selects the
    top-k records."""
    import numpy as np
    import torch

    import paper_1210_0461_b200 as crop
    from paper_1210_0461_b200 import kernels

    dev = torch.device("cuda", torch.cuda.current_device())
    hasher = crop.make_hashes(crop.HashConfig(cfg.kappa, crop.derive_seed(0, "instance:0")))
    tables = kernels.hash_tables(hasher, cfg.n_items)
    host_off = dtx.offsets.cpu().numpy()
    flush = torch.empty(1 << 28, dtype=torch.int32, device=dev)
    n_tx = dtx.n_tx
    chunks = [(t0, min(n_tx, t0 + STREAM_CHUNK_TX)) for t0 in range(0, n_tx, STREAM_CHUNK_TX)]

    def step(ev=None):
        s = kernels.StreamingSummaries(cfg.kappa, cfg.ss_capacity, tables)
        loads = torch.zeros(cfg.kappa, dtype=torch.int64, device=dev)
        for k, (t0, t1) in enumerate(chunks):
            if ev is not None:
                ev[k][0].record()
            ent = kernels.count_pairs(dtx.slice(t0, t1, host_off), True)
            if ev is not None:
                ev[k][1].record()
            bl, _, _ = kernels.entry_bucket_stats(ent, [tables], cfg.kappa, cfg.n_items, None)
            loads += bl[0]
            s.absorb(ent)
            del ent
        rec = kernels.DeviceEntries(s.row, s.col, s.count, None, s.n, 0)
        idx = kernels.topk_indices(rec, cfg.top_k)
        return s, loads, (rec.row[idx], rec.col[idx], rec.count[idx])

    sampler = ClockSampler(torch.cuda.current_device())  # started before the warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = kernels.launch_counter()
    times, count_ms = [], []
    with sampler:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in chunks]
            e0.record()
            s, loads, top = step(ev)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            count_ms.append(sum(a.elapsed_time(b) for a, b in ev))
    launches = kernels.launch_counter() - launches0
    ms = statistics.mean(times)
    lens = (dtx.offsets[1:] - dtx.offsets[:-1])
    terms = int((lens * (lens - 1) // 2).sum().item())
    bucket_loads = [int(x) for x in loads.cpu().tolist()]
    assert sum(bucket_loads) == terms
    balance = {"partitions": cfg.kappa,
               "max_mean": crop.LoadReport(kappa=cfg.kappa, workers=cfg.kappa, rows=[bucket_loads],
                                           input_pair_total=0).max_avg_ratio(),
               "max_terms": max(bucket_loads), "mean_terms": sum(bucket_loads) / cfg.kappa,
               "source": "exact per-bucket term counts of the chunks (LoadReport.max_avg_ratio arithmetic)"}
    in_bytes = 4 * int(dtx.items.numel()) + 8 * int(dtx.offsets.numel())
    summary_bytes = s.state_bytes()
    # B_alg: 8 B per term + input + the kappa * l * 16 B summaries
    b_alg = 8 * terms + in_bytes + cfg.kappa * cfg.ss_capacity * 16
    peak, peak_src = peaks()
    achieved = b_alg / (ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": "per chunk of 8.3e6 transactions: pair engine (k_item_terms, "
                "k_plan_coop, k_stream_count, k_stream_write, k_count_stream, k_reduce_slabs) -> crop_ss_index + "
                "crop_ss_probe + crop_ss_append + crop_bucket_topk + crop_ss_keep (summary merge)",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": b_alg, "avg_launch_ms": round(ms, 3),
                "phases": {"count": {"ms": round(statistics.mean(count_ms), 3),
                                     "share_of_step": round(statistics.mean(count_ms) / ms, 4)},
                           "merge": {"ms": round(ms - statistics.mean(count_ms), 3),
                                     "share_of_step": round(1 - statistics.mean(count_ms) / ms, 4)}},
                "mode": f"streaming summaries, {len(chunks)} chunks"}
    e2e = None if args.no_e2e else run_e2e_streaming(args, cfg, dtx, terms)
    cpu = None if args.no_cpu else cpu_baseline(args, cfg, dtx)
    line = {
        "metric": BASELINE_METRIC, "value": terms / (ms * 1e-3), "unit": "terms/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic: seeded Zipf transactions (SURVEY.md §8d, data seed = config no.)",
        "config": config_dict(cfg, 1),
        "details": {"terms": terms, "chunks": len(chunks), "summary_records": s.n,
                    "summary_bytes": summary_bytes, "summary_bound_bytes": cfg.kappa * cfg.ss_capacity * 16,
                    "peak_device_bytes": int(torch.cuda.max_memory_allocated())},
        "partition_balance": balance, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(launches), "clocks": sampler.summary(),
    }
    print(json.dumps(line), flush=True)


def run_e2e_streaming(args, cfg, dtx, terms):
    """Public API end to end: pinned host transactions -> crop.run_streaming
    -> SketchState.top_entries(top_k) + every summary record to pinned host
    memory (SketchState.entry_arrays)."""
    import numpy as np
    import torch

    import paper_1210_0461_b200 as crop

    off_h = dtx.offsets.cpu().pin_memory()
    it_h = dtx.items.cpu().pin_memory()
    off_np, it_np = off_h.numpy(), it_h.numpy().view(np.uint32)
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=cfg.ss_capacity, workers=cfg.workers,
                               cs_enabled=False, seed=0)
    out = [None]
    d2h = [0]

    def once():
        stream = crop.TransactionStream(cfg.n_items, off_np, it_np, validate=False)
        state, report = crop.run_streaming(stream, config, upper_triangle_only=True,
                                           chunk_transactions=STREAM_CHUNK_TX)
        top = state.top_entries(cfg.top_k)
        if out[0] is None:
            tdt = {np.uint16: torch.int16, np.uint32: torch.int32}
            out[0] = tuple(torch.empty(cfg.kappa * cfg.ss_capacity, dtype=tdt[dt], pin_memory=True)
                           .numpy().view(dt) for dt in (*state.entry_dtypes()[:1] * 2, state.entry_dtypes()[1]))
        row, col, cnt = state.entry_arrays(out=out[0])
        per = row.dtype.itemsize + col.dtype.itemsize + cnt.dtype.itemsize
        d2h[0] = cfg.kappa * 8 + cfg.top_k * 32 + per * int(row.shape[0])
        torch.cuda.synchronize()
        return top

    once()
    times = []
    for _ in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        once()
        times.append(time.perf_counter() - t0)
    tm = statistics.mean(times)
    return {"value": terms / tm, "unit": "terms/s", "ms_per_step": tm * 1e3,
            "h2d_bytes_per_step": off_h.numel() * 8 + it_h.numel() * 4, "d2h_bytes_per_step": d2h[0],
            "api": "crop.run_streaming(TransactionStream) + SketchState.top_entries + "
                   "SketchState.entry_arrays (every summary record to pinned host memory)"}


def run_product(args, rank, world):
    """c4: real-valued C = A*B, entries hashed to kappa buckets; rank r owns the
    bucket interval split(kappa, N)[r] (the reference's worker intervals)."""
    import numpy as np
    import torch

    import paper_1210_0461_b200 as crop
    from paper_1210_0461_b200 import kernels, workloads

    cfg = workloads.CONFIGS[args.config]
    dev = torch.device("cuda", torch.cuda.current_device())
    s = workloads.generate_product_workload(cfg)  # same seed on every rank: no broadcast needed
    ds = kernels.DeviceOuterStream.from_host(s)
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.kappa,
                               cs_enabled=False, seed=0)
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, config.instance_seeds()[0]))
    tab = kernels.hash_tables(h, cfg.n)
    asg = crop.WorkerAssignment.split(cfg.kappa, world)[rank]
    flush = torch.empty(1 << 28, dtype=torch.int32, device=dev)
    total_terms = int((np.diff(s.a_ptr) * np.diff(s.b_ptr)).sum())

    def step():
        return kernels.outer_product(ds, False, cfg.kappa, asg.start, asg.stop, *tab)

    sampler = ClockSampler(torch.cuda.current_device())  # started before the warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = kernels.launch_counter()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    times = []
    with sampler:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ent = step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    launches = kernels.launch_counter() - launches0
    t_sum = sum(times)
    if world > 1:
        t = torch.tensor([t_sum], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_sum = float(t.item())
    ms = t_sum / args.steps
    own_terms = ent.total_terms if world == 1 else None
    # B_alg: 8 B per term + input (8 B per nnz per side +
    # pointers) + output (row, col u32, value f64, bucket u32 = 20 B per entry)
    nnz = int(s.a_idx.shape[0] + s.b_idx.shape[0])
    in_bytes = 12 * nnz + 16 * (s.length + 1)
    b_alg = 8 * ent.total_terms + in_bytes + 20 * ent.n
    peak, peak_src = peaks()
    achieved = b_alg / (statistics.mean(times) * 1e-3) / 1e9
    e2e = None if args.no_e2e else product_e2e(args, cfg, s, rank, world, total_terms)
    if rank == 0:
        line = {
            "metric": BASELINE_METRIC, "value": total_terms / (ms * 1e-3), "unit": "terms/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded Pareto-nnz CSC/CSR, N(0,1) fp32 values (SURVEY.md §8d)",
            "config": config_dict(cfg, world),
            "details": {"buckets_per_gpu": f"split(kappa={cfg.kappa}, {world})[rank]",
                        "terms": total_terms, "entries": ent.n if world == 1 else None},
            "roofline": {"bound": "hbm", "kernel": "scan (all-term offsets) -> k_nnz_hash -> k_bm_hist -> "
                         "k_bm_colscan -> scan (partition offsets) -> k_bm_scatter -> k_bm_sort "
                         "(bucket-major partitions sorted in shared memory, ordered fp64 run "
                         "sums, look-back output offsets)",
                         "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.config),
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": b_alg,
                         "avg_launch_ms": round(statistics.mean(times), 4)},
            "cpu_baseline": (product_cpu_baseline(args, cfg, s) if world == 1 and not args.no_cpu
                             else None),
            "e2e": e2e,
            "gpu_launches": int(launches), "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)


def product_e2e(args, cfg, s, rank, world, total_terms):
    """Public API from pinned host buffers, every step: H2D of A (CSC) and B
    (CSR), crop.partition_product for this rank's bucket interval, and the
    D2H of every entry (row, col, value, bucket) into pinned host arrays."""
    import numpy as np
    import torch

    import paper_1210_0461_b200 as crop

    def pin(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    host = [pin(x) for x in (s.a_ptr, s.a_idx, s.a_val, s.b_ptr, s.b_idx, s.b_val)]
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=world,
                               cs_enabled=False, seed=0)
    out = None
    d2h = [0]

    def once():
        nonlocal out
        st = crop.ColumnRowStream(cfg.n, cfg.n, *host)
        part = crop.partition_product(st, config, worker=rank if world > 1 else None)
        n = len(part)
        if out is None or out[0].shape[0] < n:
            cap = int(n * 1.05) + 1024
            out = tuple(torch.empty(cap, dtype=dt, pin_memory=True).numpy().view(nd)
                        for dt, nd in ((torch.int32, np.uint32), (torch.int32, np.uint32),
                                       (torch.float32, np.float32)))
        # c4 (BASELINE): sorted COO per partition, fp32 values within rel 1e-5 /
        # abs 1e-6 of the float64 reference: each exact fp64 sum is rounded once;
        # the partitions are contiguous, so their offsets replace a bucket column
        row, col, val, ptr = part.arrays(out=out, value_dtype=np.float32, bucket_ptr=True)
        d2h[0] = 12 * int(row.shape[0]) + 8 * int(ptr.shape[0])
        torch.cuda.synchronize()

    for _ in range(max(2, args.warmup // 2)):
        once()
    times = []
    for _ in range(max(1, min(args.steps, 5))):
        t0 = time.perf_counter()
        once()
        times.append(time.perf_counter() - t0)
    tm = statistics.mean(times)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([tm], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tm = float(t.item())
    h2d = sum(int(x.nbytes) for x in host)
    return {"value": total_terms / tm, "unit": "terms/s", "ms_per_step": tm * 1e3,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h[0],
            "api": "crop.partition_product(ColumnRowStream) + ProductPartition.arrays(value_dtype=float32, "
                   "bucket_ptr=True) (every entry (row, col, fp32 value) and the partition offsets to "
                   "pinned host memory)"}


def product_cpu_baseline(args, cfg, s, n_products=None):
    """The reference's per-partition enumerate_interval + fp64 dict
    accumulation (interval.py:236-254, engine.py:584-591), restated in C
    (oracle run_parallel, exact regime): shared-nothing worker intervals of
    the kappa buckets on all host cores, over the first products."""
    import numpy as np

    import oracle
    import paper_1210_0461_b200 as crop

    k = min(n_products or args.cpu_sample_tx or 100_000, s.length)
    a1, b1 = int(s.a_ptr[k]), int(s.b_ptr[k])
    st = oracle.Stream(s.a_ptr[: k + 1], s.a_idx[:a1], s.a_val[:a1],
                       s.b_ptr[: k + 1], s.b_idx[:b1], s.b_val[:b1])
    terms = int((np.diff(s.a_ptr[: k + 1]) * np.diff(s.b_ptr[: k + 1])).sum())
    cores = cpu_count()
    workers = min(cores, cfg.kappa)
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, crop.derive_seed(0, "instance:0")))
    t0 = time.perf_counter()
    oracle.run_parallel(st, h.coefficients(), cfg.kappa, workers, capacity=0, upper_only=False,
                        threads=workers)
    t = time.perf_counter() - t0
    return {"value": terms / t, "unit": "terms/s", "cores": workers, "kind": "port",
            "sample": f"first {k} of {s.length} products ({terms} terms), per-partition "
                      f"enumerate_interval + fp64 dict restatement, {workers} shared-nothing "
                      f"workers (bucket intervals of kappa={cfg.kappa}) on {workers} threads",
            "seconds": round(t, 3)}


def run_e2e(args, cfg, dtx, rank, world):
    """Public API from pinned host buffers, every step: H2D of the input,
    crop.run (count), SketchState.top_entries, and the D2H of EVERY counted
    entry (row, col, support) into pinned host arrays
    (SketchState.entry_arrays) -- c2 "report all counts"."""
    import numpy as np
    import torch

    import paper_1210_0461_b200 as crop

    off_h = dtx.offsets.cpu().pin_memory()
    # the host stream holds uint16 item ids when the universe fits (c2, c5):
    # TransactionStream keeps them and the upload moves half the bytes
    small = cfg.n_items <= 65536
    it_h = (dtx.items.to(torch.int16) if small else dtx.items).cpu().pin_memory()
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.workers,
                               cs_enabled=False, seed=0)
    off_np, it_np = off_h.numpy(), it_h.numpy().view(np.uint16 if small else np.uint32)
    out = None
    d2h = [0]

    def once():
        nonlocal out
        stream = crop.TransactionStream(cfg.n_items, off_np, it_np, validate=False)
        if world > 1:
            from paper_1210_0461_b200 import distributed

            top, report = distributed.top_entries_distributed(stream if rank == 0 else None,
                                                              config, cfg.top_k)
            d2h[0] = cfg.kappa * 8 + cfg.top_k * 24
        else:
            state, report = crop.run(stream, config, upper_triangle_only=True)
            top = state.top_entries(cfg.top_k)
            n = state.device_result.entries.n
            if out is None or out[0].shape[0] < n:
                cap = int(n * 1.05) + 1024
                idt, wdt = state.entry_dtypes()
                tdt = {np.uint16: torch.int16, np.uint32: torch.int32}
                out = tuple(torch.empty(cap, dtype=tdt[dt], pin_memory=True).numpy().view(dt)
                            for dt in (idt, idt, wdt))
            row, col, cnt = state.entry_arrays(out=out)
            # loads (kappa u64) + top-k + every entry's (row, col, count)
            per = row.dtype.itemsize + col.dtype.itemsize + cnt.dtype.itemsize
            d2h[0] = cfg.kappa * 8 + cfg.top_k * 24 + per * int(row.shape[0])
        torch.cuda.synchronize()
        return report

    for _ in range(max(2, args.warmup // 2)):
        once()
    times = []
    for _ in range(max(1, min(args.steps, 5))):
        t0 = time.perf_counter()
        report = once()
        times.append(time.perf_counter() - t0)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([max(times)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tm = float(t.item())
    else:
        tm = statistics.mean(times)
    terms = int(((dtx.offsets[1:] - dtx.offsets[:-1]) *
                 (dtx.offsets[1:] - dtx.offsets[:-1] - 1) // 2).sum().item())
    h2d = off_h.numel() * 8 + it_h.numel() * it_h.element_size()
    return {"value": terms / tm, "unit": "terms/s", "ms_per_step": tm * 1e3,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h[0],
            "api": "crop.run(TransactionStream, uint16 item ids when the universe fits) + "
                   "SketchState.top_entries + SketchState.entry_arrays (all counts to pinned host memory)"
            if world == 1 else "distributed.top_entries_distributed"}


def default_sample(cfg_name):
    # about 10 s of oracle work on the box's host threads
    return {"c1": 20_000, "c2": 500_000, "c3": 400_000, "c5": 10_000, "c4": 100_000}.get(
        cfg_name, 50_000)


def cpu_baseline(args, cfg, dtx):
    """C oracle (reference algorithm restated) on a bounded prefix of the
    workload, all host cores."""
    n_sample = args.cpu_sample_tx or default_sample(args.config)
    n_sample = min(n_sample, dtx.n_tx)
    off = dtx.offsets[: n_sample + 1].cpu().numpy()
    items = dtx.items[: int(off[-1])].cpu().numpy().view("uint32")
    return cpu_baseline_arrays(args, cfg, off, items)


def cpu_baseline_arrays(args, cfg, off, items):
    import numpy as np

    import oracle
    import paper_1210_0461_b200 as crop

    n_sample = off.shape[0] - 1
    lens = np.diff(off)
    terms = int((lens * (lens - 1) // 2).sum())
    cores = cpu_count()
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, crop.derive_seed(0, "instance:0")))
    stream = oracle.Stream(off, items)
    t0 = time.perf_counter()
    oracle.run_parallel(stream, h.coefficients(), cfg.kappa, cfg.workers, capacity=0,
                        upper_only=True, threads=cores)
    t = time.perf_counter() - t0
    return {"value": terms / t, "unit": "terms/s", "cores": min(cores, cfg.workers),
            "kind": "port",
            "sample": f"first {n_sample} of {cfg.n_tx} transactions ({terms} terms), "
                      f"run_parallel restatement: {cfg.workers} shared-nothing workers "
                      f"on {min(cores, cfg.workers)} threads, exact summaries",
            "seconds": round(t, 3)}


# ------------------------------------------------------------------ reference arm

def host_workload_sample(cfg, n_tx):
    """The first n_tx transactions of the config's seeded workload, built on
    the host by the oracle's copy of the generator (no product library)."""
    import oracle
    from paper_1210_0461_b200 import workloads

    alias = workloads.zipf_alias(cfg.n_items, cfg.zipf_s)
    cdf, lo = workloads.length_cdf(cfg.length)
    return oracle.gen_transactions(n_tx, cfg.n_items, alias, cdf, lo, cfg.seed)


def run_reference(args, rank, world):
    """The reference algorithm on the host cores (the reference package is pure
    Python and absent on the GPU box: its C restatement, oracle/, stands in;
    kind "port"). Rank 0 alone; no CUDA context, no product library."""
    if rank != 0:
        return
    from paper_1210_0461_b200 import workloads

    cfg = workloads.CONFIGS[args.config]
    if not isinstance(cfg, workloads.PairConfig):
        s = workloads.generate_product_workload(cfg)  # numpy, host
        vals = [product_cpu_baseline(args, cfg, s) for _ in range(args.warmup + args.steps)]
        vals = vals[args.warmup:]
        dtype = "f64"
        data = "synthetic: seeded Pareto-nnz CSC/CSR, N(0,1) fp32 values (SURVEY.md §8d)"
    else:
        n_sample = args.cpu_sample_tx or default_sample(args.config)
        off, items = host_workload_sample(cfg, min(n_sample, cfg.n_tx))
        vals = []
        for k in range(args.warmup + args.steps):
            r = cpu_baseline_arrays(args, cfg, off, items)
            if k >= args.warmup:
                vals.append(r)
        dtype = "u32"
        data = "synthetic: seeded Zipf transactions (SURVEY.md §8d, data seed = config no.)"
    value = statistics.mean(v["value"] for v in vals)
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": value, "unit": "terms/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(v["seconds"] for v in vals) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype,
        "data": data, "config": config_dict(cfg, world),
        "cpu_baseline": {"value": value, "unit": "terms/s", "cores": vals[0]["cores"],
                         "kind": "port", "sample": vals[0]["sample"]},
        "e2e": {"value": value, "unit": "terms/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)  # host only: rank 0 runs, the others exit 0
        return
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
