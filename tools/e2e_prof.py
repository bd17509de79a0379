"""Stage timing of the public-API end-to-end path on c2 (dev tool)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import engine, workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dtx = workloads.generate_pairs_workload(cfg)
off_h = dtx.offsets.cpu().pin_memory()
it_h = dtx.items.cpu().pin_memory()
off_np, it_np = off_h.numpy(), it_h.numpy().view(np.uint32)
config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.workers, cs_enabled=False, seed=0)


def tick(label, t, log):
    torch.cuda.synchronize()
    now = time.perf_counter()
    log.append((label, (now - t) * 1e3))
    return now


for it in range(4):
    log = []
    t = t0 = time.perf_counter()
    stream = crop.TransactionStream(cfg.n_items, off_np, it_np, validate=False)
    t = tick("stream", t, log)
    prep = engine.prepare(stream)
    t = tick("prepare (H2D, n_items, pair total)", t, log)
    result, _ = engine._compute(prep, config, True)
    t = tick("compute (tables, count, stats)", t, log)
    result.finalize_summaries()
    t = tick("finalize", t, log)
    state = crop.SketchState._from_device(config, prep.n_rows, prep.n_cols, True, result)
    top = state.top_entries(cfg.top_k)
    t = tick("top_entries", t, log)
    print(f"iter {it}: total {(t - t0) * 1e3:.2f} ms  " + "  ".join(f"{k} {v:.2f}" for k, v in log))
