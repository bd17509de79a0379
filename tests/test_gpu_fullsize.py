"""Full-size BASELINE configurations on one B200: size-independent properties.

The oracle cannot finish c2 / c3 / c5 / c4 at full size in test time (SURVEY.md
§8c), so the CUDA path is checked at those sizes through properties that do
not depend on the size, against independent computations:

* conservation: the counts sum to the workload's term count;
* per-bucket loads of the counted entries == the independent bucket-load
  kernel (`count_sorted` restatement, crop_selfjoin_bucket_loads);
* keys are unique (every pair counted in exactly one place);
* spot recounts: the top entries and random entries recounted from the
  inverted item -> transaction lists with plain torch ops (no project kernel);
* tile shards (the multi-GPU split) are disjoint and cover the whole job;
* c4 (real-valued): linearity sum(C) == sum_k sum(a_k) * sum(b_k), and random
  entries recomputed in float64 on the host (tolerance rel 1e-5 / abs 1e-6).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402


def _terms(dtx):
    lens = dtx.offsets[1:] - dtx.offsets[:-1]
    return int((lens * (lens - 1) // 2).sum().item())


def _keys(ent):
    return ((ent.row[: ent.n].to(torch.int64) & 0xFFFFFFFF) << 32) | (
        ent.col[: ent.n].to(torch.int64) & 0xFFFFFFFF)


class _Inverted:
    """item -> ascending transaction ids, from torch.sort (independent recount)."""

    def __init__(self, dtx):
        lens = dtx.offsets[1:] - dtx.offsets[:-1]
        owner = torch.repeat_interleave(torch.arange(dtx.n_tx, device=lens.device, dtype=torch.int32),
                                        lens)
        items = dtx.items.to(torch.int64)
        order = torch.sort(items, stable=True).indices
        self.tx = owner[order]
        self.start = torch.searchsorted(items[order], torch.arange(dtx.n_items + 1, device=lens.device))

    def support(self, i, j):
        a = self.tx[self.start[i]: self.start[i + 1]]
        b = self.tx[self.start[j]: self.start[j + 1]]
        return int(torch.isin(a, b).sum().item())


def _check_pairs_full(name, n_spot=24):
    cfg = workloads.CONFIGS[name]
    dtx = workloads.generate_pairs_workload(cfg)
    terms = _terms(dtx)
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.workers,
                               cs_enabled=False, seed=0)
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, config.instance_seeds()[0]))
    hr, hc = kernels.hash_tables(h, cfg.n_items)
    ent = kernels.count_pairs(dtx, True)
    assert ent.total_terms == terms
    cnt = ent.count[: ent.n].to(torch.int64)
    assert int(cnt.sum().item()) == terms                      # conservation
    assert int(cnt.min().item()) >= 1
    keys = _keys(ent)
    sk = torch.sort(keys).values
    assert bool((sk[1:] > sk[:-1]).all().item())               # unique keys
    assert bool((ent.row[: ent.n] < ent.col[: ent.n]).all().item())  # upper triangle
    # per-bucket loads: counted entries vs the independent load kernel
    loads, _, _ = kernels.entry_bucket_stats(ent, [(hr, hc)], cfg.kappa, cfg.n_items, None)
    want = kernels.selfjoin_bucket_loads(dtx, hr, hc, cfg.kappa, True)
    assert torch.equal(loads[0].to(torch.int64).cpu(), want.cpu())
    # spot recounts: top entries and random entries
    inv = _Inverted(dtx)
    idx = kernels.topk_indices(ent, n_spot)
    g = torch.Generator(device="cpu").manual_seed(cfg.seed)
    rnd = torch.randint(0, ent.n, (n_spot,), generator=g).to(ent.row.device)
    for k in torch.cat([idx, rnd]).tolist():
        i, j, c = int(ent.row[k]), int(ent.col[k]), int(ent.count[k])
        assert inv.support(i, j) == c, (i, j, c)
    # the k-th largest count bounds every count outside the top-k
    top = ent.count[idx].to(torch.int64)
    mask = torch.ones(ent.n, dtype=torch.bool, device=cnt.device)
    mask[idx] = False
    assert int(cnt[mask].max().item()) <= int(top.min().item())
    return dtx, ent, cnt


def test_c2_full_size_properties():
    _check_pairs_full("c2")


def test_c5_full_size_properties_and_shards():
    dtx, ent, cnt = _check_pairs_full("c5", n_spot=8)
    # items 0 and 1 are in (nearly) every transaction at s = 1.5: top support
    assert int(cnt.max().item()) <= dtx.n_tx
    whole = torch.sort(_keys(ent))
    wcnt = cnt[whole.indices]
    wkeys = whole.values
    del ent, cnt
    # 8 tile shards: disjoint, covering, same counts (the 8-GPU split)
    parts_k, parts_c = [], []
    for r in range(8):
        job = kernels.PairCountJob(dtx, True, None, shard=(r, 8))
        e = job.run()
        job.close()
        parts_k.append(_keys(e))
        parts_c.append(e.count[: e.n].to(torch.int64))
        del e
    keys = torch.cat(parts_k)
    order = torch.sort(keys)
    assert torch.equal(order.values, wkeys)
    assert torch.equal(torch.cat(parts_c)[order.indices], wcnt)


def _row_terms(dtx):
    """Terms per row item (pairs (i, j > i)) from the positions, plain torch."""
    want = torch.zeros(dtx.n_items, dtype=torch.int64, device=dtx.offsets.device)
    step = 5_000_000
    for t0 in range(0, dtx.n_tx, step):
        off = dtx.offsets[t0: min(dtx.n_tx, t0 + step) + 1]
        lens = off[1:] - off[:-1]
        base = torch.repeat_interleave(off[:-1], lens)
        L = torch.repeat_interleave(lens, lens)
        g = torch.arange(int(off[0]), int(off[-1]), device=off.device, dtype=torch.int64)
        want.index_add_(0, dtx.items[int(off[0]): int(off[-1])].to(torch.int64), L - 1 - (g - base))
    return want


def _unique_keys(ent):
    # torch.sort is limited to 2^31 - 1 elements: check row classes mod 4
    for q in range(4):
        sel = (ent.row[: ent.n] & 3) == q
        k = torch.sort(_keys(ent)[sel]).values
        assert bool((k[1:] > k[:-1]).all().item())
        del k, sel


def test_c3_full_size_shard_conservation():
    """c3 (5e7 transactions, 1e6 items, 2.25e10 terms) as 8 tile shards run one
    after the other: every shard's keys are unique, and the counts of all
    shards sum, row by row, to the terms of each row item (rows 0-4 sit in
    more than 2^24 transactions)."""
    cfg = workloads.CONFIGS["c3"]
    dtx = workloads.generate_pairs_workload(cfg)
    want = _row_terms(dtx)
    assert int(want.sum().item()) == _terms(dtx)
    got = torch.zeros_like(want)
    for r in range(8):
        e = kernels.count_pairs_shard(dtx, True, None, shard=(r, 8), capacity=1_500_000_000)
        _unique_keys(e)
        got.index_add_(0, e.row[: e.n].to(torch.int64), e.count[: e.n].to(torch.int64))
        del e
        torch.cuda.empty_cache()
    assert torch.equal(got, want)


def test_c4_full_size_linearity_and_spot_entries():
    cfg = workloads.CONFIGS["c4"]
    s = workloads.generate_product_workload(cfg)
    ds = kernels.DeviceOuterStream.from_host(s)
    ent = kernels.outer_product(ds, False)
    assert ent.total_terms == int((np.diff(s.a_ptr) * np.diff(s.b_ptr)).sum())
    # linearity: sum of all entries of C = sum_k (sum a_k)(sum b_k)
    owner_a = np.repeat(np.arange(s.length), np.diff(s.a_ptr))
    owner_b = np.repeat(np.arange(s.length), np.diff(s.b_ptr))
    sa = np.bincount(owner_a, weights=s.a_val, minlength=s.length)
    sb = np.bincount(owner_b, weights=s.b_val, minlength=s.length)
    want = float((sa * sb).sum())
    got = float(ent.value[: ent.n].sum().item())
    scale = float((np.bincount(owner_a, weights=np.abs(s.a_val), minlength=s.length) *
                   np.bincount(owner_b, weights=np.abs(s.b_val), minlength=s.length)).sum())
    assert abs(got - want) <= 1e-6 + 1e-12 * scale  # fp64 sums of the same fp32 values
    # random entries recomputed on the host in float64
    rows = ent.row[: ent.n]
    cols = ent.col[: ent.n]
    g = torch.Generator(device="cpu").manual_seed(4)
    pick = torch.randint(0, ent.n, (16,), generator=g).tolist()
    for k in pick:
        i, j, v = int(rows[k]), int(cols[k]), float(ent.value[k])
        ka = owner_a[s.a_idx == i]
        va = s.a_val[s.a_idx == i]
        kb = owner_b[s.b_idx == j]
        vb = s.b_val[s.b_idx == j]
        common, ia, ib = np.intersect1d(ka, kb, return_indices=True)
        ref = float((va[ia] * vb[ib]).sum())
        assert abs(v - ref) <= 1e-6 + 1e-5 * abs(ref), (i, j, v, ref)
