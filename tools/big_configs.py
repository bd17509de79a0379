"""Full-size c3 / c5 on one B200: whole job or one rank's tile shard (dev tool).

    python tools/big_configs.py c5 [world] [ranks] [capacity]

Prints per-iteration CUDA-event time, phases, terms, entries and the
conservation check (sum of counts == terms of the shard) for each rank.
"""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ranks = [int(r) for r in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
cap = int(float(sys.argv[4])) if len(sys.argv) > 4 else None
cfg = workloads.CONFIGS[name]
t0 = time.perf_counter()
dtx = workloads.generate_pairs_workload(cfg)
torch.cuda.synchronize()
lens = dtx.offsets[1:] - dtx.offsets[:-1]
terms_all = int((lens * (lens - 1) // 2).sum().item())
print(f"{name}: n_tx={dtx.n_tx} nnz={dtx.nnz} terms={terms_all:.4e} gen={time.perf_counter() - t0:.1f}s",
      flush=True)
config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.workers,
                           cs_enabled=False, seed=0)
h = crop.make_hashes(crop.HashConfig(cfg.kappa, config.instance_seeds()[0]))
tab = kernels.hash_tables(h, cfg.n_items)
tot = 0
for r in ranks:
    iters = int(os.environ.get("ITERS", "3"))
    for it in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        try:
            job = kernels.PairCountJob(dtx, True, None, keep=tab, shard=(r, G))
        except crop.ResourceCapError:
            ent = kernels.count_pairs_shard(dtx, True, None, keep=tab, shard=(r, G), capacity=cap)
            e1.record()
            torch.cuda.synchronize()
            n = ent.n
            ms = e0.elapsed_time(e1)
            print(f"  rank {r}/{G} it{it}: {ms:.3f} ms in {ent.sub_shards} sub-shards entries={n}", flush=True)
            if it < iters - 1:
                del ent
            continue
        job.set_timing(True)
        ent = job.run(sync=False, capacity=cap)
        e1.record()
        torch.cuda.synchronize()
        n = int(ent.n_dev.item())
        ph = job.phase_ms()
        ms = e0.elapsed_time(e1)
        mode = job.stream_mode
        info = (job.total_terms, job.n_tiles, job.n_units, job.max_entries)
        ov = job.overflowed()
        job.close()
        print(f"  rank {r}/{G} it{it}: {ms:.3f} ms mode={'stream' if mode else 'entry'} "
              f"entries={n} cap={ent.capacity} overflow={ov or n > ent.capacity} "
              f"phases={ {k: round(v, 3) for k, v in ph.items()} } info={info}", flush=True)
        if it < iters - 1:
            del ent
            torch.cuda.empty_cache()
    if cfg.ss_capacity and n <= ent.capacity:
        ent.n = n
        times = []
        for _ in range(3):
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record()
            mask, bmin, btot = kernels.bucket_topk(ent, tab[0], tab[1], cfg.kappa, cfg.ss_capacity)
            b1.record()
            torch.cuda.synchronize()
            times.append(round(b0.elapsed_time(b1), 3))
        print(f"  rank {r}: per-bucket top-{cfg.ss_capacity} summaries {min(times):.3f} ms (runs {times}), "
              f"recorded {int(mask.sum())}, full buckets {int((btot >= cfg.ss_capacity).sum())}", flush=True)
        del mask
    if n <= ent.capacity:
        s = int(ent.count[:n].to(torch.int64).sum().item())
        mx = int(ent.count[:n].max().item())
        tot += s
        print(f"  rank {r}: sum(counts)={s} max={mx} terms/s={s / (ms * 1e-3):.3e}", flush=True)
    del ent
    torch.cuda.empty_cache()
print(f"sum over ranks {ranks}: {tot} (all terms {terms_all}) "
      f"{'CONSERVED' if len(ranks) == G and tot == terms_all else ''}")
print(f"max mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")
