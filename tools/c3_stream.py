"""c3 on one GPU through the streaming summaries (crop.run_streaming's loop,
timed per phase): chunk count, absorb, summary bytes (dev tool).
Usage: python tools/c3_stream.py [n_tx] [chunk_tx]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

cfg = workloads.CONFIGS["c3"]
n_tx = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n_tx
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 5_000_000
t = time.perf_counter()
dtx = workloads.generate_pairs_workload(cfg, n_tx=n_tx)
torch.cuda.synchronize()
print(f"generated {n_tx} tx, {dtx.nnz} items in {time.perf_counter() - t:.1f} s", flush=True)
h = crop.make_hashes(crop.HashConfig(cfg.kappa, crop.derive_seed(0, "instance:0")))
tab = kernels.hash_tables(h, cfg.n_items)
host_off = dtx.offsets.cpu().numpy()
for rep in range(2):
    s = kernels.StreamingSummaries(cfg.kappa, cfg.ss_capacity, tab)
    tc = ta = 0.0
    terms = 0
    peak = 0
    torch.cuda.reset_peak_memory_stats()
    t_all = time.perf_counter()
    for t0 in range(0, n_tx, chunk):
        t1 = min(n_tx, t0 + chunk)
        torch.cuda.synchronize()
        a = time.perf_counter()
        ent = kernels.count_pairs(dtx.slice(t0, t1, host_off), True)
        torch.cuda.synchronize()
        b = time.perf_counter()
        s.absorb(ent)
        torch.cuda.synchronize()
        c = time.perf_counter()
        tc += b - a
        ta += c - b
        terms += ent.total_terms
        print(f"  chunk [{t0}, {t1}): {ent.n} entries, count {1e3 * (b - a):.1f} ms, absorb {1e3 * (c - b):.1f} ms, "
              f"records {s.n}, candidates {getattr(s, 'last_candidates', 0)}", flush=True)
        del ent
    tot = time.perf_counter() - t_all
    print(f"rep {rep}: total {tot:.2f} s (count {tc:.2f}, absorb {ta:.2f}) -> {terms / tot:.3e} terms/s; "
          f"summary bytes {s.state_bytes() / 1e9:.3f} GB (kappa*l*16 = {cfg.kappa * cfg.ss_capacity * 16 / 1e9:.3f} GB); "
          f"peak device memory {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
