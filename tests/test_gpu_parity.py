"""GPU parity: the CUDA path (through the public API / C-ABI) against the
reference's golden fixtures and the C oracle on the same seeded inputs.

Integer work (hashes, buckets, loads, pair counts, Count-Sketch cells of 0/1
streams, top-k order) must match bit for bit; real-valued products are summed
in fp64 in stream order and must match bit for bit as well (tolerance
rel 1e-5 / abs 1e-6 is what BASELINE.json allows; we assert exact equality).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1210_0461_b200 as crop  # noqa: E402
from conftest import tx_to_csr, vectors_to_csr  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402


def _records(recs):
    return sorted((int(b), int(r), int(c), float(n), float(o)) for b, r, c, n, o in recs)


def _state_records(state):
    out = []
    for inst in state.instances:
        rs = []
        for b, s in inst.summaries.items():
            for item, cnt, over in s.records():
                rs.append((b, item[0], item[1], cnt, over))
        out.append(sorted(rs))
    return out


# ----------------------------------------------------------------- hashing

def test_device_hash_tables_match_reference(golden):
    for case in golden["hashes"]:
        h = crop.make_hashes(crop.HashConfig(case["kappa"], case["seed"]))
        assert list(h.coefficients()) == case["coeffs"]
        idx = case["indices"]
        n = max(idx) + 1
        if n > (1 << 24):
            continue  # tables for huge ids are checked through index_hash below
        hr, hc = kernels.hash_tables(h, n)
        hr = kernels.u32_to_numpy(hr)
        hc = kernels.u32_to_numpy(hc)
        assert hr[idx].tolist() == case["h_row"]
        assert hc[idx].tolist() == case["h_col"]


def test_device_sign_hash(golden):
    for case in golden["hashes"]:
        h = crop.make_hashes(crop.HashConfig(case["kappa"], case["seed"]))
        rows = torch.tensor([r for r, _, _ in case["signs"]], dtype=torch.int64).to(torch.int32)
        cols = torch.tensor([c for _, c, _ in case["signs"]], dtype=torch.int64).to(torch.int32)
        s = kernels.sign_hash(rows.cuda(), cols.cuda(), h.sign_hash).cpu().tolist()
        assert s == [x for _, _, x in case["signs"]]


# ----------------------------------------------------------------- mining golden

@pytest.mark.parametrize("case_idx", range(5))
def test_run_matches_reference_golden(golden, case_idx):
    case = golden["mining"][case_idx]
    cfg = crop.EngineConfig(**case["config"])
    stream = crop.transactions_to_stream(case["transactions"])
    state, report = crop.run(stream, cfg, upper_triangle_only=True)
    assert report.rows == case["rows"]
    assert report.input_pair_total == case["input_pair_total"]
    assert report.assignments == [tuple(a) for a in case["assignments"]]
    assert report.max_avg_ratio() == case["max_avg_ratio"]
    exact = cfg.ss_capacity >= 2 ** 31
    for inst, want in zip(state.instances, case["instances"]):
        assert inst.seed == want["seed"]
        assert list(inst.hasher.coefficients()) == want["coeffs"]
        assert inst.sketch.cells == want["cs"]
        for b, tot in want["bucket_totals"].items():
            assert inst.summaries[int(b)].total_weight == tot
    if exact:
        got = _state_records(state)
        for g, want in zip(got, case["instances"]):
            assert g == _records(want["records"])
        top = [[t.entry.row, t.entry.col, t.lower, t.upper, t.estimate]
               for t in state.top_entries(25)]
        assert top == case["top25"]
        for i, j, lo, up, est in case["queries"]:
            assert list(state.query((i, j))) == [lo, up, est]
    else:
        # bounded regime: Space-Saving guarantees against exact supports
        supports = {(a, b): c for a, b, c in case["supports"]}
        for inst in state.instances:
            for b, s in inst.summaries.items():
                m = s.total_weight
                for item, cnt, over in s.records():
                    assert cnt - over <= supports[item] <= cnt
                    assert over <= m / cfg.ss_capacity
        for (i, j), true in supports.items():
            lo, up, _ = state.query((i, j))
            assert lo <= true <= up


def test_measure_loads_matches_reference(golden):
    for case in golden["mining"]:
        cfg = crop.EngineConfig(**case["config"])
        stream = crop.transactions_to_stream(case["transactions"])
        up = crop.measure_loads(stream, cfg, upper_triangle_only=True)
        full = crop.measure_loads(stream, cfg, upper_triangle_only=False)
        assert up.rows == case["loads_upper"]
        assert full.rows == case["loads_full"]
        assert full.input_pair_total == case["pair_total_full"]


def test_selfjoin_full_matches_reference(golden):
    case = golden["selfjoin_full"]
    cfg = crop.EngineConfig(**case["config"])
    stream = crop.transactions_to_stream(case["transactions"])
    state, report = crop.run(stream, cfg, upper_triangle_only=False)
    assert report.rows == case["rows"]
    got = _state_records(state)
    assert got[0] == _records(case["instances"][0]["records"])
    assert state.instances[0].sketch.cells == case["instances"][0]["cs"]


def test_exact_pair_supports_matches_reference(golden):
    for case in golden["mining"]:
        got = crop.exact_pair_supports(case["transactions"])
        assert sorted([a, b, c] for (a, b), c in got.items()) == case["supports"]


# ----------------------------------------------------------------- general streams

def _general_stream(case):
    ap, ai, av = vectors_to_csr(case["a"])
    bp, bi, bv = vectors_to_csr(case["b"])
    return crop.ColumnRowStream(case["n_dim"], case["n_dim"], ap, ai, av, bp, bi, bv)


def test_exact_product_matches_reference(golden):
    for case in golden["general"]:
        s = _general_stream(case)
        got = crop.exact_product(s)
        assert sorted([a, b, w] for (a, b), w in got.items()) == case["exact"]
        got = crop.exact_product(s, upper_only=True)
        assert sorted([a, b, w] for (a, b), w in got.items()) == case["exact_upper"]


def test_partition_enumeration_matches_reference(golden):
    for case in golden["general"]:
        s = _general_stream(case)
        h = crop.make_hashes(crop.HashConfig(case["kappa"], case["seed"]))
        ds = kernels.DeviceOuterStream.from_host(s)
        tab = kernels.hash_tables(h, case["n_dim"])
        for part in case["partitions"]:
            ent = kernels.outer_product(ds, False, case["kappa"], part["start"], part["stop"], *tab)
            r, c, w = ent.to_numpy()
            assert sorted([int(a), int(b), float(x)] for a, b, x in zip(r, c, w)) == part["entries"]
            loads = kernels.outer_bucket_loads(ds, tab[0], tab[1], case["kappa"], False)
            assert int(loads[part["start"]:part["stop"]].sum()) == part["count"]


def test_enumerate_interval_single_products(golden):
    case = golden["general"][1]
    h = crop.make_hashes(crop.HashConfig(case["kappa"], case["seed"]))
    for (ai, av), (bi, bv) in list(zip(case["a"], case["b"]))[:6]:
        a = crop.SparseVector(case["n_dim"], ai, av)
        b = crop.SparseVector(case["n_dim"], bi, bv)
        for asg in crop.WorkerAssignment.split(case["kappa"], case["workers"]):
            got = list(crop.enumerate_interval(a, b, h.row_hash, h.col_hash, asg))
            want = [((i, j), a.get(i) * b.get(j)) for i in ai for j in bi
                    if asg.start <= h.bucket_of(i, j) < asg.stop]
            assert sorted((tuple(e), v) for e, v in got) == sorted(want)
            assert crop.count_interval(a, b, h.row_hash, h.col_hash, asg) == len(want)


def test_run_rejects_negative_terms(golden):
    s = _general_stream(golden["general"][0])
    with pytest.raises(crop.InputError):
        crop.run(s, crop.EngineConfig(kappa=4, ss_capacity=8))


# ----------------------------------------------------------------- config workloads vs oracle

def _oracle_pairs(off, items):
    r, c, w = oracle.pair_supports(off, items)
    return oracle.sorted_pairs(r, c, w)


def _gpu_pairs(ent):
    r, c, w = ent.to_numpy()
    return oracle.sorted_pairs(r, c, w)


@pytest.fixture(params=["auto", "entry", "stream", "stream-host-plan"])
def count_mode(request, monkeypatch):
    """Counting mode of the pair engine: the planner's choice, or forced;
    stream mode with the device planner (default) or the host planner."""
    if request.param == "entry":
        monkeypatch.setenv("CROP_FORCE_ENTRY_MODE", "1")
    elif request.param.startswith("stream"):
        monkeypatch.setenv("CROP_FORCE_STREAM_MODE", "1")
    if request.param.endswith("host-plan"):
        monkeypatch.setenv("CROP_HOST_PLANNER", "1")
    return request.param


@pytest.mark.parametrize("name,n_tx", [("c1", None), ("c2", 60_000), ("c5", 3_000),
                                       ("c3", 30_000)])
def test_config_prefix_counts_bit_exact(name, n_tx, count_mode):
    cfg = workloads.CONFIGS[name]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=n_tx)
    off, items = dtx.to_host()
    ent = kernels.count_pairs(dtx, True)
    gr, gc, gw = _gpu_pairs(ent)
    orow, ocol, ow = _oracle_pairs(off, items)
    assert np.array_equal(gr, orow) and np.array_equal(gc, ocol) and np.array_equal(gw, ow)
    lens = np.diff(off)
    assert ent.total_terms == int((lens * (lens - 1) // 2).sum())
    assert int(gw.sum()) == ent.total_terms  # conservation


def test_c1_full_run_against_oracle():
    cfg = workloads.CONFIGS["c1"]
    dtx = workloads.generate_pairs_workload(cfg)
    off, items = dtx.to_host()
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.workers, seed=0)
    state, report = crop.run(dtx, config, upper_triangle_only=True)
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, config.instance_seeds()[0]))
    recs, loads = oracle.run(oracle.Stream(off, items), h.coefficients(), cfg.kappa, cfg.workers,
                             upper_only=True, cs=True)
    assert report.rows[0] == loads.tolist()
    assert state.device_result.instances[0].cs.tolist() == recs.cs.tolist()
    top = state.top_entries(cfg.top_k)
    want = sorted(zip(recs.count.tolist(), recs.row.tolist(), recs.col.tolist()),
                  key=lambda x: (-x[0], x[1], x[2]))[: cfg.top_k]
    assert [(t.entry.row, t.entry.col, t.upper) for t in top] == [(r, c, n) for n, r, c in want]


@pytest.mark.parametrize("kappa,workers,worker", [(8, 8, 3), (1184, 8, 5), (16, 4, 0)])
def test_interval_filter_matches_oracle_worker(kappa, workers, worker, count_mode):
    cfg = workloads.CONFIGS["c2"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=20_000)
    off, items = dtx.to_host()
    config = crop.EngineConfig(kappa=kappa, ss_capacity=2 ** 31, workers=workers, seed=7)
    h = crop.make_hashes(crop.HashConfig(kappa, config.instance_seeds()[0]))
    asg = config.assignments()[worker]
    tab = kernels.hash_tables(h, cfg.n_items)
    ent = kernels.count_pairs(dtx, True, kappa, asg.start, asg.stop, *tab)
    recs, load = oracle.run_worker(oracle.Stream(off, items), h.coefficients(), kappa, workers,
                                   worker, upper_only=True)
    want = oracle.sorted_pairs(recs.row, recs.col, recs.count)
    got = _gpu_pairs(ent)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    assert int(got[2].sum()) == load


def test_mine_fimi_file_matches_oracle(tmp_path):
    """crop.mine over a FIMI file (native reader -> GPU) equals the oracle."""
    cfg = workloads.CONFIGS["c1"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=5000)
    off, items = dtx.to_host()
    path = tmp_path / "c1.dat"
    with open(path, "w") as fh:
        for k in range(off.shape[0] - 1):
            fh.write(" ".join(str(x) for x in items[off[k]:off[k + 1]].tolist()) + "\n")
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.workers,
                               cs_enabled=True, seed=0)
    state, report = crop.mine(path, config)
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, config.instance_seeds()[0]))
    recs, loads = oracle.run(oracle.Stream(off, items), h.coefficients(), cfg.kappa, cfg.workers,
                             upper_only=True, cs=True)
    assert report.rows[0] == loads.tolist()
    g = _gpu_pairs(state.device_result.entries)
    o = oracle.sorted_pairs(recs.row, recs.col, recs.count)
    for x, y in zip(g, o):
        assert np.array_equal(x, y)


def test_small_output_capacity_reruns():
    """An output capacity below the distinct count is detected and re-run."""
    cfg = workloads.CONFIGS["c2"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=20_000)
    off, items = dtx.to_host()
    job = kernels.PairCountJob(dtx, True, None)
    try:
        ent = job.run(capacity=1000)
    finally:
        job.close()
    assert ent.n > 1000 and ent.row.shape[0] >= ent.n
    g = _gpu_pairs(ent)
    o = _oracle_pairs(off, items)
    for x, y in zip(g, o):
        assert np.array_equal(x, y)


def test_mode_choice():
    """Short transactions (c2) count in stream mode, long ones (c5) in entry mode."""
    for name, n_tx, want in (("c2", 20_000, True), ("c5", 2_000, False)):
        dtx = workloads.generate_pairs_workload(workloads.CONFIGS[name], n_tx=n_tx)
        job = kernels.PairCountJob(dtx, True, None)
        assert job.stream_mode is want
        job.close()


def test_topk_with_ties_matches_sort():
    cfg = workloads.CONFIGS["c2"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=30_000)
    ent = kernels.count_pairs(dtx, True)
    r, c, w = ent.to_numpy()
    order = np.lexsort((c, r, -w))
    for k in (1, 7, 1000, 5000, int(r.shape[0]), int(r.shape[0]) + 10):
        idx = kernels.topk_indices(ent, k).cpu().numpy()
        got = sorted(zip(-w[idx], r[idx], c[idx]))
        want = sorted(zip(-w[order[:k]], r[order[:k]], c[order[:k]]))
        assert got == want


def test_c4_prefix_product_matches_oracle():
    cfg = workloads.CONFIGS["c4"]
    s = workloads.generate_product_workload(cfg, n_products=20_000)
    s = crop.ColumnRowStream(cfg.n, cfg.n, s.a_ptr, s.a_idx, s.a_val, s.b_ptr, s.b_idx, s.b_val)
    ds = kernels.DeviceOuterStream.from_host(s)
    h = crop.make_hashes(crop.HashConfig(cfg.kappa, crop.derive_seed(0, "instance:0")))
    tab = kernels.hash_tables(h, cfg.n)
    ent = kernels.outer_product(ds, False, cfg.kappa, 0, cfg.kappa, *tab)
    gr, gc, gw = ent.to_numpy()
    ost = oracle.Stream(s.a_ptr, s.a_idx, s.a_val, s.b_ptr, s.b_idx, s.b_val)
    orow, ocol, ow = oracle.exact_product(ost)
    # include exact zero sums on the GPU side for comparison
    nz = gw != 0.0
    g = oracle.sorted_pairs(gr[nz], gc[nz], gw[nz])
    o = oracle.sorted_pairs(orow, ocol, ow)
    assert np.array_equal(g[0], o[0]) and np.array_equal(g[1], o[1])
    np.testing.assert_allclose(g[2], o[2], rtol=1e-5, atol=1e-6)
    assert np.array_equal(g[2], o[2])  # stream-ordered fp64 sums: bit-exact
    # per-bucket sorted COO
    b = kernels.u32_to_numpy(ent.bucket[: ent.n])
    assert np.all(np.diff(b.astype(np.int64)) >= 0)
    key = (b.astype(np.uint64) << np.uint64(40)) | (gr.astype(np.uint64) << np.uint64(20)) | gc
    assert np.all(np.diff(key.astype(np.int64)) > 0)


def test_edge_cases():
    # empty stream, empty and singleton transactions
    for tx in ([], [[]], [[5]], [[], [1, 2], [3]], [[0, 1, 2, 3]]):
        stream = crop.transactions_to_stream(tx, dim=8)
        cfg = crop.EngineConfig(kappa=3, ss_capacity=100, workers=3, seed=1)
        state, report = crop.run(stream, cfg, upper_triangle_only=True)
        sup = {}
        for t in tx:
            for a in range(len(t)):
                for b in range(a + 1, len(t)):
                    sup[(t[a], t[b])] = sup.get((t[a], t[b]), 0) + 1
        assert report.total_entries == sum(sup.values())
        for (i, j), v in sup.items():
            assert state.query((i, j))[:2] == (v, v)
        assert len(state.top_entries(5)) == min(5, len(sup))


def test_row_with_more_than_2_24_occurrences(count_mode):
    """A row item in more than 2^24 transactions (c3's heaviest rows have
    4.4e7): its occurrence count must survive pass A's packing, or the units
    are sized too few and the 16-bit counters wrap."""
    n_tx = (1 << 24) + (1 << 20)
    offsets = np.arange(0, 2 * n_tx + 1, 2, dtype=np.int64)
    items = np.empty(2 * n_tx, dtype=np.uint32)
    items[0::2] = 0
    items[1::2] = 1 + (np.arange(n_tx) % 64)
    dtx = kernels.DeviceTransactions.from_host(offsets, items, 65)
    ent = kernels.count_pairs(dtx, True)
    r, c, w = ent.to_numpy()
    got = dict(zip(zip(r.tolist(), c.tolist()), w.tolist()))
    want = np.bincount(np.arange(n_tx) % 64, minlength=64)
    assert got == {(0, j + 1): float(want[j]) for j in range(64)}


def test_long_transactions_and_wide_rows(count_mode):
    # lengths up to the 8192 limit; n > kDenseCap forces column windows
    rng = np.random.default_rng(0)
    n = 120_000
    tx = [np.unique(rng.integers(0, n, size=L)).tolist() for L in (8000, 300, 5000, 2)]
    tx += [[0, 1, 2, n - 1], [0, n - 2, n - 1]] * 20
    # a row with > kHashCap terms and > kDenseCap columns -> column windows
    tx += [[0] + np.unique(rng.integers(1, n, size=1000)).tolist() for _ in range(30)]
    off, items = tx_to_csr(tx)
    dtx = kernels.DeviceTransactions.from_host(off, items, n)
    ent = kernels.count_pairs(dtx, True)
    g = _gpu_pairs(ent)
    o = _oracle_pairs(off, items)
    for x, y in zip(g, o):
        assert np.array_equal(x, y)
    too_long = [list(range(9000))]
    off, items = tx_to_csr(too_long)
    with pytest.raises(crop.InputError):
        kernels.count_pairs(kernels.DeviceTransactions.from_host(off, items, 9000), True)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_host_generator_copy_matches_device_generator(name):
    """bench.py's reference arm builds its sample with the oracle's host copy
    of the generator (no product library); it must be the same data."""
    cfg = workloads.CONFIGS[name]
    n = 20_000
    dtx = workloads.generate_pairs_workload(cfg, n_tx=n)
    off, items = oracle.gen_transactions(n, cfg.n_items, workloads.zipf_alias(cfg.n_items, cfg.zipf_s),
                                         *workloads.length_cdf(cfg.length), cfg.seed)
    d_off, d_items = dtx.to_host()
    assert np.array_equal(off, d_off)
    assert np.array_equal(items, d_items)


def test_uint16_item_ids_give_the_same_run():
    """A TransactionStream built from uint16 item ids keeps them (half the
    upload) and counts exactly what the uint32 stream counts."""
    cfg = workloads.CONFIGS["c1"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=3000)
    off, items = dtx.to_host()
    config = crop.EngineConfig(kappa=4, ss_capacity=2 ** 31, workers=4, cs_enabled=False, seed=0)
    s32 = crop.TransactionStream(cfg.n_items, off, items)
    s16 = crop.TransactionStream(cfg.n_items, off, items.astype(np.uint16))
    assert s16.items.dtype == np.uint16 and s32.items.dtype == np.uint32
    a, ra = crop.run(s32, config, upper_triangle_only=True)
    b, rb = crop.run(s16, config, upper_triangle_only=True)
    assert ra.rows == rb.rows
    ea, eb = a.entry_arrays(), b.entry_arrays()
    assert sorted(zip(*(x.tolist() for x in ea))) == sorted(zip(*(x.tolist() for x in eb)))
    assert a.top_entries(20) == b.top_entries(20)
    with pytest.raises(crop.InputError):
        crop.TransactionStream(10, off, items.astype(np.uint16))  # ids outside the universe


@pytest.mark.parametrize("compact", [True, False])
def test_entry_arrays_columns(compact):
    """SketchState.entry_arrays: every counted entry with its support, as
    uint16 ids when both dimensions fit (compact) or uint32, into caller
    buffers of the named dtypes or fresh pinned arrays; equal to the oracle."""
    cfg = workloads.CONFIGS["c1"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=3000)
    off, items = dtx.to_host()
    stream = crop.TransactionStream(cfg.n_items, off, items)
    config = crop.EngineConfig(kappa=4, ss_capacity=2 ** 31, workers=4, cs_enabled=False, seed=0)
    state, _ = crop.run(stream, config, upper_triangle_only=True)
    idt, wdt = state.entry_dtypes(compact)
    assert idt == (np.uint16 if compact else np.uint32) and wdt == np.uint32
    row, col, w = state.entry_arrays(compact=compact)
    assert row.dtype == idt and col.dtype == idt and w.dtype == np.uint32
    er, ec, ew = oracle.pair_supports(off, items)
    want = sorted(zip(er.tolist(), ec.tolist(), ew.astype(np.int64).tolist()))
    assert sorted(zip(row.tolist(), col.tolist(), w.tolist())) == want
    n = row.shape[0]
    out = (np.empty(n + 5, idt), np.empty(n + 5, idt), np.empty(n + 5, wdt))
    r2, c2, w2 = state.entry_arrays(out=out, compact=compact)
    assert np.array_equal(r2, row) and np.array_equal(c2, col) and np.array_equal(w2, w)
    # transfers on the copy stream under other device work: valid after wait_entries()
    out3 = tuple(torch.empty(n, dtype={2: torch.int16, 4: torch.int32}[np.dtype(dt).itemsize],
                             pin_memory=True).numpy().view(dt) for dt in (idt, idt, wdt))
    r3, c3, w3 = state.entry_arrays(out=out3, compact=compact, wait=False)
    top = state.top_entries(10)
    state.wait_entries()
    assert np.array_equal(r3, row) and np.array_equal(c3, col) and np.array_equal(w3, w)
    assert len(top) == 10
    with pytest.raises(crop.InputError):
        state.entry_arrays(out=(np.empty(n, np.uint64), np.empty(n, np.uint64), np.empty(n, np.uint64)),
                           compact=compact)
