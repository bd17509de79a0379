"""Host-side timing of the pieces of crop.run + top_entries on c2 (dev tool)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import engine, kernels, workloads  # noqa: E402

cfg = workloads.CONFIGS["c2"]
dtx = workloads.generate_pairs_workload(cfg)
off_h = dtx.offsets.cpu().pin_memory()
it_h = dtx.items.cpu().pin_memory()
off_np, it_np = off_h.numpy(), it_h.numpy().view(np.uint32)
config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.workers, cs_enabled=False, seed=0)


def tick(log, label, t):
    torch.cuda.synchronize()
    now = time.perf_counter()
    log.append((label, (now - t) * 1e3))
    return now


for it in range(5):
    log = []
    t = t0 = time.perf_counter()
    stream = crop.TransactionStream(cfg.n_items, off_np, it_np, validate=False)
    prep = engine.prepare(stream)
    t = tick(log, "prepare", t)
    seeds = config.instance_seeds()
    hashers = [crop.make_hashes(crop.HashConfig(config.kappa, s)) for s in seeds]
    t = tick(log, "make_hashes", t)
    tables = [kernels.hash_tables(h, prep.n_items) for h in hashers]
    t = tick(log, "hash_tables", t)
    job = kernels.PairCountJob(prep.device, True, None)
    t = tick(log, "create", t)
    ent = job.run()
    t = tick(log, "run", t)
    job.close()
    loads, distinct, cs = kernels.entry_bucket_stats(ent, [tables[0]], config.kappa, prep.n_items, None)
    t = tick(log, "bucket_stats", t)
    l0, d0 = loads[0].cpu().numpy(), distinct[0].cpu().numpy()
    t = tick(log, "stats.cpu", t)
    idx = kernels.topk_indices(ent, cfg.top_k)
    t = tick(log, "topk_indices", t)
    parts = [ent.row[idx], ent.col[idx], ent.count[idx]]
    h = torch.stack([p.to(torch.int64) for p in parts]).cpu().numpy()
    t = tick(log, "gather+d2h", t)
    order = np.lexsort((h[1], h[0], -h[2]))
    res = [(int(a), int(b), int(c)) for a, b, c in zip(h[0][order], h[1][order], h[2][order])]
    t = tick(log, "host sort+list", t)
    print(f"iter {it}: total {(t - t0) * 1e3:.2f} ms  " + "  ".join(f"{k} {v:.3f}" for k, v in log), flush=True)
    del ent
