"""Randomised parity of the pair engine (GPU) against the C oracle.

Seeded random streams across the engine's regimes: tiny and wide item
universes (ids >= 2^16 disable the 16-bit item copy; > 57,344 columns force
column windows), empty / singleton / long transactions, skewed and uniform
ids, upper-triangle and full self-joins, whole and partial bucket intervals,
and each counting mode. Counts must be bit-exact (the oracle restates the
reference's exact regime, pinned by tests/test_oracle_golden.py).
"""

import numpy as np
import pytest

import oracle
import paper_1210_0461_b200 as crop
from paper_1210_0461_b200 import kernels

pytestmark = pytest.mark.gpu


def _stream(rng, n_tx, n_items, max_len, skew):
    rows = []
    for _ in range(n_tx):
        L = int(rng.integers(0, max_len + 1))
        if skew:
            ids = np.minimum((rng.pareto(1.1, size=L) * 3).astype(np.int64), n_items - 1)
        else:
            ids = rng.integers(0, n_items, size=L)
        rows.append(np.unique(ids))
    lens = np.array([r.shape[0] for r in rows], dtype=np.int64)
    off = np.zeros(n_tx + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    items = np.concatenate(rows).astype(np.uint32) if n_tx else np.zeros(0, np.uint32)
    return off, items


CASES = []
_r = np.random.default_rng(12345)
for case in range(80):
    n_items = int(_r.choice([3, 60, 2500, 30000, 70000]))
    n_tx = int(_r.choice([1, 40, 700, 3000, 20000]))
    CASES.append(dict(
        seed=case, n_items=n_items, n_tx=n_tx,
        max_len=int(_r.choice([1, 4, 30] if n_tx > 3000 else [1, 4, 30, 300])),
        skew=bool(_r.integers(0, 2)),
        upper=bool(_r.integers(0, 4) > 0),
        kappa=int(_r.choice([1, 8, 16])),
        mode=str(_r.choice(["auto", "entry", "stream"]))))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"s{c['seed']}-n{c['n_items']}-{c['mode']}")
def test_random_streams_bit_exact(case, monkeypatch):
    if case["mode"] == "entry":
        monkeypatch.setenv("CROP_FORCE_ENTRY_MODE", "1")
    elif case["mode"] == "stream":
        monkeypatch.setenv("CROP_FORCE_STREAM_MODE", "1")
    rng = np.random.default_rng(case["seed"])
    off, items = _stream(rng, case["n_tx"], case["n_items"], case["max_len"], case["skew"])
    kappa = case["kappa"]
    workers = min(4, kappa)
    worker = int(rng.integers(0, workers))
    h = crop.make_hashes(crop.HashConfig(kappa, crop.derive_seed(case["seed"], "instance:0")))
    asg = crop.WorkerAssignment.split(kappa, workers)[worker]
    dtx = kernels.DeviceTransactions.from_host(off, items, case["n_items"])
    tab = kernels.hash_tables(h, case["n_items"])
    ent = kernels.count_pairs(dtx, case["upper"], kappa, asg.start, asg.stop, *tab)
    gr, gc, gw = oracle.sorted_pairs(*ent.to_numpy())
    recs, load = oracle.run_worker(oracle.Stream(off, items), h.coefficients(), kappa, workers,
                                   worker, upper_only=case["upper"])
    orow, ocol, ow = oracle.sorted_pairs(recs.row, recs.col, recs.count)
    assert np.array_equal(gr, orow) and np.array_equal(gc, ocol) and np.array_equal(gw, ow)
    assert int(gw.sum()) == load


@pytest.mark.parametrize("name,n_tx,world,mode", [("c2", 50_000, 3, "auto"), ("c2", 50_000, 8, "auto"),
                                                   ("c5", 2_000, 3, "auto"), ("c2", 30_000, 4, "entry"),
                                                   ("c3", 20_000, 5, "stream")])
def test_tile_shards_partition_the_job(name, n_tx, world, mode, monkeypatch):
    """The ranks' tile shards are disjoint and together equal the whole job."""
    from paper_1210_0461_b200 import workloads

    if mode == "entry":
        monkeypatch.setenv("CROP_FORCE_ENTRY_MODE", "1")
    elif mode == "stream":
        monkeypatch.setenv("CROP_FORCE_STREAM_MODE", "1")
    dtx = workloads.generate_pairs_workload(workloads.CONFIGS[name], n_tx=n_tx)
    off, items = dtx.to_host()
    parts = []
    for r in range(world):
        job = kernels.PairCountJob(dtx, True, None, shard=(r, world))
        try:
            ent = job.run()
        finally:
            job.close()
        parts.append(ent.to_numpy())
    row = np.concatenate([p[0] for p in parts])
    col = np.concatenate([p[1] for p in parts])
    w = np.concatenate([p[2] for p in parts])
    key = row.astype(np.int64) << 32 | col.astype(np.int64)
    assert np.unique(key).shape[0] == key.shape[0]  # disjoint
    g = oracle.sorted_pairs(row, col, w)
    o = oracle.sorted_pairs(*oracle.pair_supports(off, items))
    for x, y in zip(g, o):
        assert np.array_equal(x, y)
