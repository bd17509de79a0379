"""Per-rank phase times of tile shards on one GPU (dev tool)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ranks = [int(sys.argv[3])] if len(sys.argv) > 3 else range(G)
dtx = workloads.generate_pairs_workload(cfg)
for r in ranks:
    for it in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        job = kernels.PairCountJob(dtx, True, None, shard=(r, G))
        job.set_timing(True)
        ent = job.run()
        e1.record()
        torch.cuda.synchronize()
        ph = job.phase_ms()
        nt, nu = job.n_tiles, job.n_units
        job.close()
    print(f"G={G} rank {r}: {e0.elapsed_time(e1):.3f} ms units={nu} entries={ent.n} "
          f"write={ph['write']:.3f} count={ph['count']:.3f}")
