"""Quick timing of the pair engine on a config (dev tool; bench.py is the contract)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n_tx = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = workloads.CONFIGS[name]
t0 = time.time()
dtx = workloads.generate_pairs_workload(cfg, n_tx=n_tx)
torch.cuda.synchronize()
print(f"{name}: gen {time.time()-t0:.2f}s n_tx={dtx.n_tx} nnz={dtx.nnz}")
for it in range(4):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2 = torch.cuda.Event(enable_timing=True)
    e0.record()
    job = kernels.PairCountJob(dtx, True, None)
    e1.record()
    ent = job.run(sync=False)
    e2.record()
    torch.cuda.synchronize()
    n = int(ent.n_dev.item())
    t_plan, t_run = e0.elapsed_time(e1), e1.elapsed_time(e2)
    print(f"iter {it}: plan {t_plan:.3f} ms  run {t_run:.3f} ms  total {t_plan+t_run:.3f} ms  "
          f"terms={job.total_terms:.3e} entries={n} tiles={job.n_tiles} units={job.n_units} "
          f"max_entries={job.max_entries}  rate={job.total_terms/((t_plan+t_run)*1e-3):.3e} terms/s")
    ent.n = n
    t3 = torch.cuda.Event(enable_timing=True); t4 = torch.cuda.Event(enable_timing=True)
    t3.record()
    idx = kernels.topk_indices(ent, cfg.top_k)
    t4.record(); torch.cuda.synchronize()
    print(f"   topk {t3.elapsed_time(t4):.3f} ms k={idx.shape[0]}")
    job.close()
