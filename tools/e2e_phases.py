"""Wall-clock phases of the c2 e2e call (bench.run_e2e's once()) with
synchronisation after each phase (dev tool)."""
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
out = None
for it in range(6):
    log = []
    torch.cuda.synchronize()
    t0 = t = time.perf_counter()

    def tick(name):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        log.append(f"{name} {1e3 * (now - t):.2f}")
        t = now

    stream = crop.TransactionStream(cfg.n_items, off_np, it_np, validate=False)
    prep = engine.prepare(stream)
    tick("prepare(H2D+reduce)")
    result, _ = engine._compute(prep, config, True)
    tick("compute")
    result.finalize_summaries()
    state = crop.SketchState._from_device(config, prep.n_rows, prep.n_cols, True, result)
    tick("finalize")
    top = state.top_entries(cfg.top_k)
    tick("top_entries")
    n = state.device_result.entries.n
    if out is None or out[0].shape[0] < n:
        idt, wdt = state.entry_dtypes()
        tdt = {np.uint16: torch.int16, np.uint32: torch.int32}
        out = tuple(torch.empty(int(n * 1.05) + 1024, dtype=tdt[dt], pin_memory=True).numpy().view(dt)
                    for dt in (idt, idt, wdt))
    row, col, cnt = state.entry_arrays(out=out)
    per = row.dtype.itemsize + col.dtype.itemsize + cnt.dtype.itemsize
    tick(f"entry_arrays({per * n / 1e6:.0f} MB)")
    print(f"iter {it}: total {1e3 * (t - t0):.2f} ms | " + " | ".join(log), flush=True)
# raw copy rates
a = torch.empty(610_000_000 // 4, dtype=torch.int32, device="cuda")
h = torch.empty_like(a, device="cpu").pin_memory()
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
    d2h = time.perf_counter() - t
    t = time.perf_counter()
    a.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    h2d = time.perf_counter() - t
    print(f"raw 610 MB: D2H {610 / d2h / 1e3:.1f} GB/s, H2D {610 / h2d / 1e3:.1f} GB/s")
