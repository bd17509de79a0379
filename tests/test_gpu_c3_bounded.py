"""The c3 heavy-hitter contract on a c3 prefix, against the C oracle's exact
supports (an independent CPU count, not the device path).

BASELINE c3 asks for per-partition Space-Saving summaries whose top-10,000
pair weights are within the paper's error bound of the exact counts. Here a
prefix of the c3 workload (kappa = 1184 buckets) runs with a capacity l
scaled so that buckets overflow, and every guarantee of spacesaving.py:1-9 /
PAPER.md:142 is checked per bucket b with m_b = its term count:

* sandwich: lower <= exact <= upper for every recorded entry;
* over <= m_b / l (here over = 0: the summaries hold exact weights);
* capture: every pair with exact > m_b / l is recorded;
* the top-10,000 by upper bound equals the exact top-10,000 except for ties
  inside the bound band at rank 10,000;

both for crop.run on the whole prefix and for 8 tile shards whose per-bucket
candidates are merged (kernels.merge_bucket_summaries, the N-GPU path).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

N_TX = 100_000
CAP = 1024
TOP = 10_000


@pytest.fixture(scope="module")
def c3_prefix():
    cfg = workloads.CONFIGS["c3"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=N_TX)
    off, items = dtx.to_host()
    row, col, w = oracle.pair_supports(off, items)
    return cfg, dtx, (row.astype(np.int64), col.astype(np.int64), w.astype(np.int64))


def _keys(row, col):
    return (np.asarray(row, np.int64) << 32) | np.asarray(col, np.int64)


def _check(cfg, hasher, exact, rec_row, rec_col, rec_w, loads, bucket_min):
    er, ec, ew = exact
    kappa = cfg.kappa
    h = hasher
    hr = np.array(h.row_hash.values(range(cfg.n_items)), np.int64)
    hc = np.array(h.col_hash.values(range(cfg.n_items)), np.int64)
    eb = (hr[er] + hc[ec]) % kappa
    # loads: m_b = sum of exact supports per bucket (LoadReport units)
    m = np.bincount(eb, weights=ew, minlength=kappa).astype(np.int64)
    assert np.array_equal(m, loads)
    # sandwich with zero overestimation: recorded weights are exact
    ex = dict(zip(_keys(er, ec).tolist(), ew.tolist()))
    rk = _keys(rec_row, rec_col).tolist()
    assert all(ex[k] == w for k, w in zip(rk, rec_w.tolist()))
    # at most l records per bucket; the bound m_b / l
    rb = (hr[rec_row] + hc[rec_col]) % kappa
    per = np.bincount(rb, minlength=kappa)
    assert per.max() <= CAP
    full = np.bincount(eb, minlength=kappa) >= CAP
    assert full.sum() > kappa // 2, "the prefix must overflow most summaries"
    bound = m / CAP
    # every bucket's summary minimum (its upper bound for absent entries) is
    # within the bound: min <= m_b / l
    assert np.all(bucket_min[full] <= bound[full])
    # capture: exact > m_b / l  =>  recorded
    heavy = ew > bound[eb]
    rec_set = set(rk)
    assert all(k in rec_set for k in _keys(er[heavy], ec[heavy]).tolist())
    # query bounds of absent entries: upper = bucket minimum of a full bucket
    absent = ~np.isin(_keys(er, ec), np.array(rk, np.int64))
    assert np.all(ew[absent] <= np.where(full[eb[absent]], bucket_min[eb[absent]], 0))
    # top-10,000 identity outside the band: exact top by (w desc, row, col)
    order = np.lexsort((ec, er, -ew))[:TOP]
    kth = ew[order[-1]]
    got = np.lexsort((rec_col, rec_row, -rec_w))[:TOP]
    band = int(bound.max())
    want_strict = set(_keys(er[order], ec[order])[ew[order] > kth + band].tolist())
    got_keys = set(_keys(rec_row[got], rec_col[got]).tolist())
    assert want_strict <= got_keys


def test_c3_prefix_bounded_regime_whole_job(c3_prefix):
    cfg, dtx, exact = c3_prefix
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=CAP, workers=8, cs_enabled=False,
                               seed=0)
    state, report = crop.run(dtx, config, upper_triangle_only=True)
    d = state.device_result
    inst = d.instances[0]
    e = d.entries
    mask = inst.recorded if inst.recorded is not None else torch.ones(e.n, dtype=torch.bool,
                                                                       device=e.row.device)
    rr = kernels.u32_to_numpy(e.row[: e.n][mask]).astype(np.int64)
    rc = kernels.u32_to_numpy(e.col[: e.n][mask]).astype(np.int64)
    rw = kernels.u32_to_numpy(e.count[: e.n][mask]).astype(np.int64)
    _check(cfg, inst.hasher, exact, rr, rc, rw, inst.loads.astype(np.int64),
           inst.bucket_min.astype(np.int64))
    # the public query surface agrees on a sample of pairs
    er, ec, ew = exact
    for x in np.random.default_rng(0).choice(er.shape[0], 300, replace=False):
        lo, up, _ = state.query((int(er[x]), int(ec[x])))
        assert lo <= ew[x] <= up
    top = state.top_entries(50)
    order = np.lexsort((ec, er, -ew))[:50]
    assert [(t.entry.row, t.entry.col, t.upper) for t in top] == \
        [(int(er[x]), int(ec[x]), float(ew[x])) for x in order]


def test_c3_prefix_bounded_regime_eight_tile_shards(c3_prefix):
    cfg, dtx, exact = c3_prefix
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, crop.derive_seed(0, "instance:0")))
    tab = kernels.hash_tables(h, cfg.n_items)
    parts = [kernels.count_pairs_shard(dtx, True, None, keep=tab, shard=(r, 8)) for r in range(8)]
    cand, mask, bmin, loads, distinct = kernels.merge_bucket_summaries(parts, tab[0], tab[1],
                                                                      cfg.kappa, CAP)
    rr = kernels.u32_to_numpy(cand.row[mask]).astype(np.int64)
    rc = kernels.u32_to_numpy(cand.col[mask]).astype(np.int64)
    rw = kernels.u32_to_numpy(cand.count[mask]).astype(np.int64)
    _check(cfg, h, exact, rr, rc, rw, loads.cpu().numpy(), bmin.cpu().numpy())
    # identical records to the whole-job summaries
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=CAP, workers=8, cs_enabled=False,
                               seed=0)
    state, _ = crop.run(dtx, config, upper_triangle_only=True)
    d = state.device_result
    e = d.entries
    m2 = d.instances[0].recorded
    whole = np.sort(_keys(kernels.u32_to_numpy(e.row[: e.n][m2]),
                          kernels.u32_to_numpy(e.col[: e.n][m2])))
    assert np.array_equal(np.sort(_keys(rr, rc)), whole)
    assert np.array_equal(bmin.cpu().numpy(), d.instances[0].bucket_min.astype(np.int64))
