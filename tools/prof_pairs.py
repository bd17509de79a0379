"""One warm pair-engine run for ncu (dev tool)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = workloads.CONFIGS[name]
dtx = workloads.generate_pairs_workload(cfg)
torch.cuda.synchronize()
for it in range(iters):
    job = kernels.PairCountJob(dtx, True, None)
    ent = job.run()
    idx = kernels.topk_indices(ent, cfg.top_k)
    torch.cuda.synchronize()
    job.close()
print("done", ent.n)
