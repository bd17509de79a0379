"""One own-bucket interval job (c2, kappa 8, bucket 3) for ncu (dev tool)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
kappa = int(sys.argv[2]) if len(sys.argv) > 2 else 8
lo, hi = (int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "3,4").split(","))
dtx = workloads.generate_pairs_workload(cfg)
h = crop.make_hashes(crop.HashConfig(kappa, crop.derive_seed(0, "instance:0")))
tab = kernels.hash_tables(h, cfg.n_items)
iv = kernels.interval_struct(kappa, lo, hi, *tab)
for _ in range(2):
    job = kernels.PairCountJob(dtx, True, iv, keep=tab)
    ent = job.run()
    job.close()
torch.cuda.synchronize()
print("own", job.own, "entries", ent.n)
