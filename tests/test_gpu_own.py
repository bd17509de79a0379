"""Own-bucket (Lemma 1) enumeration of filtered pair jobs.

A job restricted to the bucket interval [start, stop) must visit only its own
terms (interval.py:125-189): its term total is the interval's load, not the
stream's, and its counts equal the oracle's run_worker restatement bit for
bit. Checked against the C oracle and against the same job without the
own-bucket layout (CROP_PAIRS_NO_OWN), over many intervals (incl. windows
that wrap around kappa), the full self-join, long transactions (every branch
of the (h_col, id) sort), the safe-unit plan and the 16-bit wrap detection.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1210_0461_b200 as crop  # noqa: E402
from conftest import tx_to_csr  # noqa: E402
from paper_1210_0461_b200 import _native as nat  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402


def _job(dtx, upper, kappa, start, stop, tab, flags=0):
    iv = kernels.interval_struct(kappa, start, stop, *tab)
    job = kernels.PairCountJob(dtx, upper, iv, keep=tab, flags=flags)
    try:
        ent = job.run()
        return ent, job.own, job.total_terms
    finally:
        job.close()


def _sorted(ent):
    r, c, w = ent.to_numpy()
    return oracle.sorted_pairs(r, c, w)


def _oracle_interval(off, items, h, kappa, start, stop, upper):
    """Counts of the entries whose bucket lies in [start, stop): the oracle's
    single-worker run restricted by bucket (run_worker over a 1-worker split
    is the whole range, so filter its records)."""
    recs, _ = oracle.run(oracle.Stream(off, items), h.coefficients(), kappa, 1, upper_only=upper)
    b = recs.bucket
    m = (b >= start) & (b < stop)
    return oracle.sorted_pairs(recs.row[m], recs.col[m], recs.count[m])


@pytest.mark.parametrize("name,n_tx,kappa,intervals", [
    ("c2", 30_000, 8, [(3, 4), (0, 1), (7, 8), (2, 6)]),
    ("c2", 30_000, 1184, [(0, 148), (1036, 1184), (500, 501), (100, 1100)]),
    ("c5", 1_500, 1184, [(148, 296), (0, 1), (1183, 1184)]),
    ("c1", None, 4, [(1, 2), (0, 3)]),
    ("c1", None, 5, [(4, 5), (2, 4)]),
])
@pytest.mark.parametrize("upper", [True, False])
def test_own_interval_matches_oracle_and_plain_filter(name, n_tx, kappa, intervals, upper):
    cfg = workloads.CONFIGS[name]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=n_tx)
    off, items = dtx.to_host()
    h = crop.make_hashes(crop.HashConfig(kappa, crop.derive_seed(11, "instance:0")))
    tab = kernels.hash_tables(h, cfg.n_items)
    for start, stop in intervals:
        ent, own, terms = _job(dtx, upper, kappa, start, stop, tab)
        assert own, "the filtered job should use the own-bucket layout"
        got = _sorted(ent)
        want = _oracle_interval(off, items, h, kappa, start, stop, upper)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)
        # only own terms were planned and routed: the job's term total is the
        # interval's load
        assert terms == int(got[2].sum())
        ent2, own2, terms2 = _job(dtx, upper, kappa, start, stop, tab, nat.PAIRS_NO_OWN)
        assert not own2
        for g, w in zip(got, _sorted(ent2)):
            assert np.array_equal(g, w)


def test_own_terms_tile_the_stream():
    """Own term totals of the K intervals of a split sum to T (every term is
    visited by exactly one interval) and equal the per-bucket loads."""
    cfg = workloads.CONFIGS["c2"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=40_000)
    lens = (dtx.offsets[1:] - dtx.offsets[:-1]).cpu().numpy()
    T = int((lens * (lens - 1) // 2).sum())
    kappa = 1184
    h = crop.make_hashes(crop.HashConfig(kappa, crop.derive_seed(0, "instance:0")))
    tab = kernels.hash_tables(h, cfg.n_items)
    loads = kernels.selfjoin_bucket_loads(dtx, tab[0], tab[1], kappa, True).cpu().numpy()
    total = 0
    for a in crop.WorkerAssignment.split(kappa, 8):
        ent, own, terms = _job(dtx, True, kappa, a.start, a.stop, tab)
        assert own
        assert terms == int(loads[a.start:a.stop].sum())
        total += terms
    assert total == T


def test_own_long_transactions_and_safe_units():
    """Transactions of <= 32, <= 2048 and > 2048 items (the three sort paths of
    k_hs_build); the safe-unit plan gives the same counts."""
    rng = np.random.default_rng(5)
    n = 20_000
    tx = [np.unique(rng.integers(0, n, size=L)).tolist() for L in (3000, 2500, 700, 64, 33, 32, 5)]
    tx += [sorted(rng.choice(n, size=rng.integers(2, 40), replace=False).tolist())
           for _ in range(4000)]
    off, items = tx_to_csr(tx)
    dtx = kernels.DeviceTransactions.from_host(off, items, n)
    kappa = 16
    h = crop.make_hashes(crop.HashConfig(kappa, 3))
    tab = kernels.hash_tables(h, n)
    for start, stop in [(5, 6), (14, 18 - 16 + 14), (0, 15)]:
        stop = min(stop, kappa)
        want = _oracle_interval(off, items, h, kappa, start, stop, True)
        for flags in (0, nat.PAIRS_SAFE_UNITS):
            ent, own, _ = _job(dtx, True, kappa, start, stop, tab, flags)
            assert own
            for g, w in zip(_sorted(ent), want):
                assert np.array_equal(g, w)


def test_counter_wrap_is_detected_and_recounted(monkeypatch):
    """A stream ordered so that one pair fills a whole unit's word range: the
    first ~600k transactions are all {0, 1} (the scatter's first wave of
    position chunks, so they claim the start of row 0's word stream), then
    1,000 long transactions give row 0 many words from few occurrences. Units
    are cut by words (~160k each, forced large with CROP_DEBUG_UNIT_TERMS), so
    pair (0, 1) would count past 65,535 in a 16-bit counter: the count kernel
    detects the wrap, the job is re-planned with safe units and the counts
    are exact."""
    rng = np.random.default_rng(1)
    n_pair = 600_000
    tx = [[0, 1]] * n_pair
    tx += [[0] + np.sort(rng.choice(np.arange(2, 5000), 1999, replace=False)).tolist()
           for _ in range(1000)]
    off, items = tx_to_csr(tx)
    n = 5000
    dtx = kernels.DeviceTransactions.from_host(off, items, n)
    kappa = 2
    h = crop.make_hashes(crop.HashConfig(kappa, 0))
    tab = kernels.hash_tables(h, n)
    b01 = h.bucket_of(0, 1)
    monkeypatch.setenv("CROP_DEBUG_UNIT_TERMS", str(1 << 40))
    iv = kernels.interval_struct(kappa, b01, b01 + 1, *tab)
    job = kernels.PairCountJob(dtx, True, iv, keep=tab)
    try:
        assert job.own
        job.run(sync=False)
        torch.cuda.synchronize()
        assert job.overflowed(), "the wrap should be detected"
    finally:
        job.close()
    ent = kernels.count_pairs(dtx, True, kappa, b01, b01 + 1, *tab)
    got = _sorted(ent)
    want = _oracle_interval(off, items, h, kappa, b01, b01 + 1, True)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    assert int(got[2][(got[0] == 0) & (got[1] == 1)][0]) == n_pair
