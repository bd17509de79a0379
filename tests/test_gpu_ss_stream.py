"""Streaming, mergeable Space-Saving (crop.run_streaming; csrc/ss_stream.cu):
bounded summary memory (kappa * l records) with the reference guarantees of
spacesaving.py:1-9 / PAPER.md:142, checked against the C oracle's exact
supports on a c3 prefix (kappa = 1184) consumed in chunks:

* sandwich: count - over <= exact <= count for every record;
* over <= m_b / l and the bucket minimum <= m_b / l;
* capture: every pair with exact > m_b / l is recorded;
* unrecorded pairs are bounded by their full bucket's minimum;
* the top-10,000 by upper bound holds the exact top-10,000 outside the band;
* at most l records per bucket: the summaries' device bytes are <= kappa*l*16.

One chunk equals the exact regime's top-l of crop.run (over = 0); small
streams with forced evictions are compared with the oracle's per-term
Space-Saving bounds and the public query / top_entries surface."""

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
    return cfg, dtx, (off, items), (row.astype(np.int64), col.astype(np.int64), w.astype(np.int64))


def _keys(row, col):
    return (np.asarray(row, np.int64) << 32) | np.asarray(col, np.int64)


def _records(state):
    d = state.device_result
    e = d.entries
    n = e.n
    r = kernels.u32_to_numpy(e.row[:n]).astype(np.int64)
    c = kernels.u32_to_numpy(e.col[:n]).astype(np.int64)
    w = kernels.u32_to_numpy(e.count[:n]).astype(np.int64)
    o = kernels.u32_to_numpy(d.over[:n]).astype(np.int64)
    return r, c, w, o, d.instances[0]


def _check_bounds(cfg, hasher, exact, rr, rc, rw, ro, loads, bmin, cap, top=TOP):
    er, ec, ew = exact
    kappa = cfg.kappa
    hr = np.array(hasher.row_hash.values(range(cfg.n_items)), np.int64)
    hc = np.array(hasher.col_hash.values(range(cfg.n_items)), np.int64)
    eb = (hr[er] + hc[ec]) % kappa
    m = np.bincount(eb, weights=ew, minlength=kappa).astype(np.int64)
    assert np.array_equal(m, loads)
    ex = dict(zip(_keys(er, ec).tolist(), ew.tolist()))
    rk = _keys(rr, rc).tolist()
    got = np.array([ex[k] for k in rk], np.int64)
    assert np.all(rw - ro <= got) and np.all(got <= rw)  # sandwich
    rb = (hr[rr] + hc[rc]) % kappa
    assert np.bincount(rb, minlength=kappa).max() <= cap
    bound = m / cap
    assert np.all(ro <= bound[rb])                      # over <= m_b / l
    assert np.all(bmin <= bound)                        # min <= m_b / l
    heavy = ew > bound[eb]
    rec = set(rk)
    assert all(k in rec for k in _keys(er[heavy], ec[heavy]).tolist())  # capture
    absent = ~np.isin(_keys(er, ec), np.array(rk, np.int64))
    assert np.all(ew[absent] <= bmin[eb[absent]])       # absent <= bucket minimum
    order = np.lexsort((ec, er, -ew))[:top]
    kth = ew[order[-1]]
    g = np.lexsort((rc, rr, -rw))[:top]
    band = int(bound.max())
    strict = set(_keys(er[order], ec[order])[ew[order] > kth + band].tolist())
    assert strict <= set(_keys(rr[g], rc[g]).tolist())
    return absent


@pytest.mark.parametrize("chunk", [7_000, 25_000])
def test_streaming_summaries_c3_prefix(c3_prefix, chunk):
    cfg, dtx, _, exact = c3_prefix
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=CAP, workers=8, cs_enabled=False, seed=0)
    state, report = crop.run_streaming(dtx, config, upper_triangle_only=True, chunk_transactions=chunk)
    rr, rc, rw, ro, inst = _records(state)
    assert ro.max() > 0, "the chunks must force evictions"
    _check_bounds(cfg, inst.hasher, exact, rr, rc, rw, ro, inst.loads.astype(np.int64),
                  inst.bucket_min.astype(np.int64), CAP)
    # summary memory: at most kappa * l records of 16 B
    assert 16 * rr.shape[0] <= cfg.kappa * CAP * 16
    # LoadReport rows equal the exact per-worker terms
    er, ec, ew = exact
    h = inst.hasher
    hr = np.array(h.row_hash.values(range(cfg.n_items)), np.int64)
    hc = np.array(h.col_hash.values(range(cfg.n_items)), np.int64)
    m = np.bincount((hr[er] + hc[ec]) % cfg.kappa, weights=ew, minlength=cfg.kappa).astype(np.int64)
    asg = config.assignments()
    assert report.rows[0] == [int(m[a.start:a.stop].sum()) for a in asg]
    # public surface: query bounds and top_entries order
    for x in np.random.default_rng(1).choice(er.shape[0], 300, replace=False):
        lo, up, _ = state.query((int(er[x]), int(ec[x])))
        assert lo <= ew[x] <= up
    top = state.top_entries(40)
    lo_all = rw - ro
    want = sorted(zip(-rw, -lo_all, rr, rc))[:40]
    assert [(t.entry.row, t.entry.col, t.upper, t.lower) for t in top] == \
        [(int(r), int(c), float(-u), float(-lo)) for u, lo, r, c in want]


def test_one_chunk_is_the_exact_top_l(c3_prefix):
    """A single chunk: the summaries are the exact regime's per-bucket top-l."""
    cfg, dtx, _, _ = c3_prefix
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=CAP, workers=8, cs_enabled=False, seed=0)
    s1, _ = crop.run_streaming(dtx, config, upper_triangle_only=True, chunk_transactions=N_TX)
    rr, rc, rw, ro, inst = _records(s1)
    assert ro.max() == 0
    s2, _ = crop.run(dtx, config, upper_triangle_only=True)
    d = s2.device_result
    e = d.entries
    m2 = d.instances[0].recorded
    whole = np.sort(_keys(kernels.u32_to_numpy(e.row[: e.n][m2]), kernels.u32_to_numpy(e.col[: e.n][m2])))
    assert np.array_equal(np.sort(_keys(rr, rc)), whole)
    assert np.array_equal(inst.bucket_min, d.instances[0].bucket_min)


@pytest.mark.parametrize("instances,cs", [(1, True), (3, False)])
def test_small_stream_many_chunks(instances, cs):
    """Tiny capacity, one transaction per chunk (the per-term limit of the
    batch update): bounds hold against the oracle's exact supports, for one
    device-backed instance and three host-materialised ones; the Count-Sketch
    cells equal the oracle's."""
    cfg = workloads.CONFIGS["c1"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=600)
    off, items = dtx.to_host()
    stream = crop.TransactionStream(cfg.n_items, off, items)
    config = crop.EngineConfig(kappa=4, ss_capacity=6, workers=2, cs_enabled=cs, instances=instances,
                               seed=11)
    state, report = crop.run_streaming(stream, config, upper_triangle_only=True, chunk_transactions=1)
    er, ec, ew = (x.astype(np.int64) for x in oracle.pair_supports(off, items))
    ex = {(int(r), int(c)): int(w) for r, c, w in zip(er, ec, ew)}
    for x in range(0, er.shape[0], 7):
        lo, up, _ = state.query((int(er[x]), int(ec[x])))
        assert lo <= ew[x] <= up
    for inst in state.instances:
        for b, summ in inst.summaries.items():
            recs = list(summ.records())
            assert len(recs) <= 6
            for item, c, over in recs:
                assert c - over <= ex[item] <= c
                assert over <= summ.total_weight / 6
    if cs:
        h = crop.make_hashes(crop.HashConfig(4, config.instance_seeds()[0]))
        recs, loads = oracle.run(oracle.Stream(off, items), h.coefficients(), 4, 2, capacity=0,
                                 upper_only=True, cs=True)
        assert state.device_result.instances[0].cs.tolist() == recs.cs.tolist()
        assert report.rows[0] == loads.tolist()
    top = state.top_entries(5)
    assert len(top) == 5 and all(t.lower <= ex[(t.entry.row, t.entry.col)] <= t.upper for t in top)


def test_streaming_rejects_real_streams():
    s = crop.ColumnRowStream(4, 4, np.array([0, 1], np.int64), np.array([1], np.uint32), np.array([2.0]),
                             np.array([0, 1], np.int64), np.array([2], np.uint32), np.array([3.0]))
    with pytest.raises(crop.ConfigError):
        crop.run_streaming(s, crop.EngineConfig(kappa=2, ss_capacity=4, workers=1, seed=0))


@pytest.mark.parametrize("kappa,cap,chunk", [(64, 100, 300), (7, 3, 50), (2048, 2, 400)])
def test_merge_with_the_cut_equals_appending_every_miss(kappa, cap, chunk):
    """The two-pass merge (per-bucket weight cut, Bloom filter in front of the
    index) keeps exactly the records of the plain batch update restated here
    in Python: hits add e, every miss becomes (mu_b + e, over mu_b), each
    bucket keeps its `cap` largest by (count desc, row, col). kappa = 2048
    takes the global-memory histograms (kappa * 16 counters exceed a CTA's
    shared memory), kappa = 64 with 100 records per bucket (6,400 records) has
    the Bloom filter on."""
    cfg = workloads.CONFIGS["c1"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=1200)
    off, items = dtx.to_host()
    h = crop.make_hashes(crop.HashConfig(kappa, crop.derive_seed(5, "instance:0")))
    tab = kernels.hash_tables(h, cfg.n_items)
    hr = np.array(h.row_hash.values(range(cfg.n_items)), np.int64)
    hc = np.array(h.col_hash.values(range(cfg.n_items)), np.int64)
    summ = kernels.StreamingSummaries(kappa, cap, tab)
    want = [dict() for _ in range(kappa)]  # bucket -> {(row, col): [count, over]}
    mu = [0] * kappa
    for t0 in range(0, dtx.n_tx, chunk):
        t1 = min(dtx.n_tx, t0 + chunk)
        ent = kernels.count_pairs(dtx.slice(t0, t1), True)
        summ.absorb(ent)
        i0, i1 = int(off[t0]), int(off[t1])
        er, ec, ew = oracle.pair_supports(off[t0:t1 + 1] - i0, items[i0:i1])
        for r, c, e in zip(er.tolist(), ec.tolist(), ew.tolist()):
            b = int((hr[r] + hc[c]) % kappa)
            rec = want[b].get((r, c))
            if rec is not None:
                rec[0] += e
            else:
                want[b][(r, c)] = [mu[b] + e, mu[b]]
        for b in range(kappa):
            if len(want[b]) >= cap:
                keep = sorted(want[b].items(), key=lambda kv: (-kv[1][0], kv[0]))[:cap]
                want[b] = dict(keep)
                mu[b] = keep[-1][1][0]
    got = sorted(zip(kernels.u32_to_numpy(summ.row).tolist(), kernels.u32_to_numpy(summ.col).tolist(),
                     kernels.u32_to_numpy(summ.count).tolist(), kernels.u32_to_numpy(summ.over).tolist()))
    exp = sorted((r, c, v[0], v[1]) for b in range(kappa) for (r, c), v in want[b].items())
    assert got == exp
    assert (summ.mu.cpu().numpy().astype(np.int64) & 0xFFFFFFFF).tolist() == mu


@pytest.mark.parametrize("ids16,pinned", [(False, True), (True, False)])
def test_staged_upload_equals_the_whole_upload(monkeypatch, ids16, pinned):
    """run_streaming's chunk-by-chunk upload of a host stream (items enqueued
    one chunk ahead on the copy stream) gives the summaries of the whole
    upload: same records, bounds, loads and top entries."""
    from paper_1210_0461_b200 import engine

    cfg = workloads.CONFIGS["c1"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=4000)
    off, items = dtx.to_host()
    if ids16:
        items = items.astype(np.uint16)
    if pinned:
        items = torch.from_numpy(items.view(np.int32)).pin_memory().numpy().view(np.uint32)
    config = crop.EngineConfig(kappa=16, ss_capacity=50, workers=4, cs_enabled=True, seed=3)

    def run():
        s = crop.TransactionStream(cfg.n_items, off, items, validate=False)
        state, report = crop.run_streaming(s, config, upper_triangle_only=True, chunk_transactions=700)
        r, c, w, o, inst = _records(state)
        return sorted(zip(r.tolist(), c.tolist(), w.tolist(), o.tolist())), report.rows, \
            inst.bucket_min.tolist(), inst.cs.tolist(), state.top_entries(30)

    whole = run()
    monkeypatch.setattr(engine, "STAGED_UPLOAD_MIN_ITEMS", 1)
    staged = run()
    assert staged == whole
