"""One counting job of a config (dev tool for ncu captures): generate the
workload, run the pair engine once (the bench's step: job + top-k), or for
c3 one streaming step (chunks + summary merges). Usage: python tools/one_job.py c5"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = workloads.CONFIGS[name]
dtx = workloads.generate_pairs_workload(cfg)
torch.cuda.synchronize()
if cfg.ss_capacity:
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, crop.derive_seed(0, "instance:0")))
    tab = kernels.hash_tables(h, cfg.n_items)
    host_off = dtx.offsets.cpu().numpy()
    chunk = -(-dtx.n_tx // 6)
    s = kernels.StreamingSummaries(cfg.kappa, cfg.ss_capacity, tab)
    for t0 in range(0, dtx.n_tx, chunk):
        ent = kernels.count_pairs(dtx.slice(t0, min(dtx.n_tx, t0 + chunk), host_off), True)
        s.absorb(ent)
        del ent
    rec = kernels.DeviceEntries(s.row, s.col, s.count, None, s.n, 0)
    kernels.topk_indices(rec, cfg.top_k)
else:
    job = kernels.PairCountJob(dtx, True, None)
    ent = job.run()
    kernels.topk_indices(ent, cfg.top_k)
    job.close()
torch.cuda.synchronize()
print("done")
