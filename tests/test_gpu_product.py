"""Real-valued partitioned products (csrc/outer.cu bucket-major path) against
the C oracle's exact_product (oracle.py:20-50 restated): per-bucket sorted
COO, fp64 sums in stream order (bit-exact; BASELINE's tolerance rel 1e-5 /
abs 1e-6 is asserted too), every bucket interval, the triangle filter,
partitions too large for shared memory (the in-CTA global-memory radix
sort), the radix-sort fallback for keys wider than 64 bits (forced with
CROP_OUTER_RADIX=1) and the public crop.partition_product surface."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1210_0461_b200 as crop  # noqa: E402
from conftest import vectors_to_csr  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402


def _want(s, h, kappa, start, stop, upper=False):
    ost = oracle.Stream(s.a_ptr, s.a_idx, s.a_val, s.b_ptr, s.b_idx, s.b_val)
    orow, ocol, ow = oracle.exact_product(ost, upper_only=upper)
    hr = np.array(h.row_hash.values(range(s.n_rows)), np.int64)
    hc = np.array(h.col_hash.values(range(s.n_cols)), np.int64)
    b = (hr[orow] + hc[ocol]) % kappa
    m = (b >= start) & (b < stop)
    order = np.lexsort((ocol[m], orow[m], b[m]))
    return orow[m][order], ocol[m][order], ow[m][order], b[m][order]


def _check(part_arrays, want):
    row, col, val, buck = part_arrays
    nz = val != 0.0  # exact_product drops exact-zero sums
    got = (row[nz], col[nz], val[nz], buck[nz])
    for g, w in zip(got, want):
        assert g.shape == w.shape
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    assert np.array_equal(got[3], want[3].astype(np.uint32))
    np.testing.assert_allclose(got[2], want[2], rtol=1e-5, atol=1e-6)
    assert np.array_equal(got[2], want[2])  # stream-ordered fp64 sums: bit-exact
    key = (buck.astype(np.uint64) << np.uint64(42)) | (row.astype(np.uint64) << np.uint64(21)) | col
    assert np.all(np.diff(key.astype(np.int64)) > 0)  # per-bucket sorted, distinct


@pytest.fixture(params=["bucket-major", "radix"])
def outer_path(request, monkeypatch):
    """Both sort paths of csrc/outer.cu: the bucket-major partition sort
    (default) and the library radix-sort fallback (CROP_OUTER_RADIX=1)."""
    if request.param == "radix":
        monkeypatch.setenv("CROP_OUTER_RADIX", "1")
    return request.param


@pytest.mark.parametrize("workers", [1, 8])
def test_partition_product_c4_prefix(workers, outer_path, monkeypatch):
    cfg = workloads.CONFIGS["c4"]
    s = workloads.generate_product_workload(cfg, n_products=30_000)
    s = crop.ColumnRowStream(cfg.n, cfg.n, s.a_ptr, s.a_idx, s.a_val, s.b_ptr, s.b_idx, s.b_val)
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=workers, seed=0,
                               cs_enabled=False)
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, config.instance_seeds()[0]))
    for w in ([None] if workers == 1 else [0, 5, 7]):
        part = crop.partition_product(s, config, worker=w)
        a = config.assignments()[0 if w is None else w]
        start, stop = (0, cfg.kappa) if w is None else (a.start, a.stop)
        _check(part.arrays(), _want(s, h, cfg.kappa, start, stop))
    # the radix-sort path gives the same arrays
    monkeypatch.setenv("CROP_OUTER_RADIX", "1")
    ref = crop.partition_product(s, config, worker=None if workers == 1 else 5).arrays()
    monkeypatch.delenv("CROP_OUTER_RADIX")
    new = crop.partition_product(s, config, worker=None if workers == 1 else 5).arrays()
    for x, y in zip(ref, new):
        assert np.array_equal(x, y)
    # compact transfer: float32 values (each fp64 sum rounded once, inside the
    # BASELINE c4 tolerance) and bucket offsets instead of the bucket column
    part = crop.partition_product(s, config, worker=None if workers == 1 else 5)
    a = config.assignments()[0 if workers == 1 else 5]
    row, col, val, buck = part.arrays()
    r32, c32, v32, ptr = part.arrays(value_dtype=np.float32, bucket_ptr=True)
    assert np.array_equal(r32, row) and np.array_equal(c32, col)
    assert v32.dtype == np.float32 and np.array_equal(v32, val.astype(np.float32))
    assert np.all(np.abs(v32.astype(np.float64) - val) <= 1e-6 + 1e-5 * np.abs(val))
    assert ptr.shape[0] == a.stop - a.start + 1 and ptr[0] == 0 and ptr[-1] == len(part)
    assert np.array_equal(np.repeat(np.arange(a.start, a.stop), np.diff(ptr)), buck.astype(np.int64))
    n = len(part)
    out = (np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.float32))
    r2, c2, v2, p2 = part.arrays(out=out, value_dtype=np.float32, bucket_ptr=True)
    assert np.array_equal(r2, row) and np.array_equal(v2, v32) and np.array_equal(p2, ptr)
    with pytest.raises(crop.InputError):
        part.arrays(out=out, value_dtype=np.float64, bucket_ptr=True)


def test_partition_product_skewed_rows(outer_path):
    """One row holding far more terms than a shared-memory partition: the
    partitions refine into column ranges of the row and stay exact."""
    rng = np.random.default_rng(2)
    n = 4000
    a, b = [], []
    for k in range(6):
        a.append(([7], [1.5 - k]))
        cols = np.sort(rng.choice(n, 3000, replace=False))
        b.append((cols.tolist(), rng.standard_normal(3000).astype(np.float32).astype(np.float64).tolist()))
    for k in range(200):
        ra = np.sort(rng.choice(n, 5, replace=False))
        cb = np.sort(rng.choice(n, 5, replace=False))
        a.append((ra.tolist(), [1.0, -2.0, 0.5, 3.0, 0.25]))
        b.append((cb.tolist(), [2.0, 1.0, -1.0, 0.5, 4.0]))
    ap, ai, av = vectors_to_csr(a)
    bp, bi, bv = vectors_to_csr(b)
    s = crop.ColumnRowStream(n, n, ap, ai, av, bp, bi, bv)
    for kappa, workers in [(1, 1), (3, 3)]:
        config = crop.EngineConfig(kappa=kappa, ss_capacity=2 ** 31, workers=workers, seed=1,
                                   cs_enabled=False)
        h = crop.make_hashes(crop.HashConfig(kappa, config.instance_seeds()[0]))
        for w in range(workers):
            a_ = config.assignments()[w]
            part = crop.partition_product(s, config, worker=w if workers > 1 else None)
            _check(part.arrays(), _want(s, h, kappa, a_.start, a_.stop))


def test_partition_product_upper_and_errors(outer_path):
    cfg = workloads.CONFIGS["c4"]
    s = workloads.generate_product_workload(cfg, n_products=5_000)
    s = crop.ColumnRowStream(cfg.n, cfg.n, s.a_ptr, s.a_idx, s.a_val, s.b_ptr, s.b_idx, s.b_val)
    config = crop.EngineConfig(kappa=16, ss_capacity=2 ** 31, workers=4, seed=3, cs_enabled=False)
    h = crop.make_hashes(crop.HashConfig(16, config.instance_seeds()[0]))
    ds = kernels.DeviceOuterStream.from_host(s)
    tab = kernels.hash_tables(h, cfg.n)
    a_ = config.assignments()[2]
    ent = kernels.outer_product(ds, True, 16, a_.start, a_.stop, *tab)
    e = ent
    arrs = (kernels.u32_to_numpy(e.row[: e.n]), kernels.u32_to_numpy(e.col[: e.n]),
            e.value[: e.n].cpu().numpy(), kernels.u32_to_numpy(e.bucket[: e.n]))
    _check(arrs, _want(s, h, 16, a_.start, a_.stop, upper=True))
    with pytest.raises(crop.ConfigError):
        crop.partition_product(s, config, worker=4)


def test_partition_product_heavy_entry(outer_path):
    """One (row, col) entry with more terms than a shared-memory partition
    holds (6,000 products share it): that partition sorts in global memory
    (stable LSD radix inside one CTA) and its sum is still in stream order."""
    rng = np.random.default_rng(5)
    n = 3000
    a, b = [], []
    for k in range(6000):
        ra = np.unique(np.concatenate([[11], rng.choice(n, 3, replace=False)]))
        cb = np.unique(np.concatenate([[29], rng.choice(n, 3, replace=False)]))
        a.append((ra.tolist(), rng.standard_normal(ra.size).astype(np.float32).astype(np.float64).tolist()))
        b.append((cb.tolist(), rng.standard_normal(cb.size).astype(np.float32).astype(np.float64).tolist()))
    ap, ai, av = vectors_to_csr(a)
    bp, bi, bv = vectors_to_csr(b)
    s = crop.ColumnRowStream(n, n, ap, ai, av, bp, bi, bv)
    for kappa, workers in [(1, 1), (4, 2)]:
        config = crop.EngineConfig(kappa=kappa, ss_capacity=2 ** 31, workers=workers, seed=2,
                                   cs_enabled=False)
        h = crop.make_hashes(crop.HashConfig(kappa, config.instance_seeds()[0]))
        for w in range(workers):
            a_ = config.assignments()[w]
            part = crop.partition_product(s, config, worker=w if workers > 1 else None)
            _check(part.arrays(), _want(s, h, kappa, a_.start, a_.stop))


def test_outer_product_edge_streams(outer_path):
    """Empty products, single-term products and an empty stream."""
    a = [([], []), ([3], [2.0]), ([0, 5], [1.0, -1.0]), ([], []), ([7], [0.5])]
    b = [([1], [1.0]), ([4], [3.0]), ([], []), ([2, 6], [1.0, 2.0]), ([7], [4.0])]
    ap, ai, av = vectors_to_csr(a)
    bp, bi, bv = vectors_to_csr(b)
    s = crop.ColumnRowStream(8, 8, ap, ai, av, bp, bi, bv)
    config = crop.EngineConfig(kappa=3, ss_capacity=2 ** 31, workers=3, seed=4, cs_enabled=False)
    h = crop.make_hashes(crop.HashConfig(3, config.instance_seeds()[0]))
    for w in range(3):
        a_ = config.assignments()[w]
        _check(crop.partition_product(s, config, worker=w).arrays(), _want(s, h, 3, a_.start, a_.stop))
    e = crop.ColumnRowStream(8, 8, np.zeros(3, np.int64), np.zeros(0, np.uint32), np.zeros(0),
                             np.zeros(3, np.int64), np.zeros(0, np.uint32), np.zeros(0))
    assert len(crop.partition_product(e, config)) == 0
