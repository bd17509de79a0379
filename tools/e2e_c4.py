"""Wall-clock phases of the c4 e2e call (bench.product_e2e's once()) with a
synchronisation after each phase, plus a cProfile of one call (dev tool)."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import workloads  # noqa: E402

cfg = workloads.CONFIGS["c4"]
s = workloads.generate_product_workload(cfg)


def pin(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


host = [pin(x) for x in (s.a_ptr, s.a_idx, s.a_val, s.b_ptr, s.b_idx, s.b_val)]
config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=1, cs_enabled=False, seed=0)
out = None


def once(log=None):
    global out
    t = time.perf_counter()
    st = crop.ColumnRowStream(cfg.n, cfg.n, *host)
    part = crop.partition_product(st, config, worker=None)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    n = len(part)
    if out is None or out[0].shape[0] < n:
        cap = int(n * 1.05) + 1024
        out = tuple(torch.empty(cap, dtype=dt, pin_memory=True).numpy().view(nd)
                    for dt, nd in ((torch.int32, np.uint32), (torch.int32, np.uint32),
                                   (torch.float32, np.float32)))
    part.arrays(out=out, value_dtype=np.float32, bucket_ptr=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if log is not None:
        log.append((1e3 * (t1 - t), 1e3 * (t2 - t1), n))


for _ in range(3):
    once()
log = []
for _ in range(5):
    once(log)
for a, b, n in log:
    print(f"partition_product {a:.2f} ms | arrays {b:.2f} ms ({12 * n / 1e6:.0f} MB)")
pr = cProfile.Profile()
pr.enable()
once()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
