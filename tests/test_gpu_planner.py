"""The cooperative stream planner (k_plan_coop, one CTA per SM) against the
single-CTA planner (CROP_PLAN_SINGLE_CTA=1): the same tiles, units and
counted entries on c1, a c2 prefix, a c3 prefix (1M items, column windows),
tile shards and a bucket-interval (own-bucket) job."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402


def _job(dtx, interval, shard, keep):
    job = kernels.PairCountJob(dtx, True, interval, keep=keep, shard=shard)
    ent = job.run()
    facts = (job.total_terms, job.n_tiles, job.n_units, job.max_entries, job.stream_mode)
    r, c, w = ent.to_numpy()
    job.close()
    order = np.lexsort((c, r))
    return facts, (r[order], c[order], w[order])


@pytest.mark.parametrize("name,n_tx", [("c1", None), ("c2", 200_000), ("c3", 60_000), ("c5", 3_000)])
def test_cooperative_planner_matches_single_cta(name, n_tx, monkeypatch):
    cfg = workloads.CONFIGS[name]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=n_tx)
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, crop.derive_seed(0, "instance:0")))
    tab = kernels.hash_tables(h, cfg.n_items)
    cases = [(None, (0, 1)), (None, (1, 4)), (None, (3, 4))]
    if cfg.kappa >= 2:
        cases.append((kernels.interval_struct(cfg.kappa, 1, 2, *tab), (0, 1)))
    for interval, shard in cases:
        monkeypatch.delenv("CROP_PLAN_SINGLE_CTA", raising=False)
        got = _job(dtx, interval, shard, tab)
        monkeypatch.setenv("CROP_PLAN_SINGLE_CTA", "1")
        want = _job(dtx, interval, shard, tab)
        assert got[0] == want[0], (name, shard, got[0], want[0])
        for x, y in zip(got[1], want[1]):
            assert np.array_equal(x, y)
