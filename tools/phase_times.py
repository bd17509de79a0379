"""Per-phase pair-engine times on a config (dev tool)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = workloads.CONFIGS[name]
dtx = workloads.generate_pairs_workload(cfg)
torch.cuda.synchronize()
for it in range(4):
    job = kernels.PairCountJob(dtx, True, None)
    job.set_timing(True)
    ent = job.run(sync=True)
    ph = job.phase_ms()
    job.close()
print(name, {k: round(v, 4) for k, v in ph.items()})
