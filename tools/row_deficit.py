"""Per-row term check of a sharded job (dev tool): which rows lose terms?

    python tools/row_deficit.py c3 8 [max_split]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = workloads.CONFIGS[name]
dtx = workloads.generate_pairs_workload(cfg)
dev = dtx.offsets.device
n = cfg.n_items
want = torch.zeros(n, dtype=torch.int64, device=dev)
occ = torch.zeros(n, dtype=torch.int64, device=dev)
step = 5_000_000
for t0 in range(0, dtx.n_tx, step):
    t1 = min(dtx.n_tx, t0 + step)
    off = dtx.offsets[t0: t1 + 1]
    lens = off[1:] - off[:-1]
    base = torch.repeat_interleave(off[:-1], lens)
    L = torch.repeat_interleave(lens, lens)
    g = torch.arange(int(off[0]), int(off[-1]), device=dev, dtype=torch.int64)
    c = L - 1 - (g - base)
    it = dtx.items[int(off[0]): int(off[-1])].to(torch.int64)
    want.index_add_(0, it, c)
    occ.index_add_(0, it, (c > 0).to(torch.int64))
    del off, lens, base, L, g, c, it
print(f"{name}: terms {int(want.sum())}", flush=True)
got = torch.zeros(n, dtype=torch.int64, device=dev)
for r in range(G):
    e = kernels.count_pairs_shard(dtx, True, None, shard=(r, G), capacity=1_500_000_000)
    rows = e.row[: e.n].to(torch.int64)
    cnt = e.count[: e.n].to(torch.int64)
    mine = torch.zeros(n, dtype=torch.int64, device=dev)
    mine.index_add_(0, rows, cnt)
    got += mine
    print(f"rank {r}: entries {e.n} terms {int(cnt.sum())} sub_shards {getattr(e, 'sub_shards', 1)} "
          f"rows {int((mine > 0).sum())}", flush=True)
    del e, rows, cnt, mine
    torch.cuda.empty_cache()
bad = torch.nonzero(got != want).flatten()
print(f"rows with wrong sums: {bad.numel()} deficit {int((want - got).sum())}")
for i in bad[:40].tolist():
    print(f"  row {i}: want {int(want[i])} got {int(got[i])} occ {int(occ[i])}")
if bad.numel():
    print(f"  first bad {int(bad.min())} last bad {int(bad.max())}")
