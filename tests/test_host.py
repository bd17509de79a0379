"""CPU tests: host logic, hashing parity, file formats, and the C-ABI surface.

No kernel is executed here (there is no GPU in the build container); the
library is loaded and its exported symbols checked against include/crop_b200.h.
"""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1210_0461_b200 as crop
from paper_1210_0461_b200 import _native, hashing, workloads
from paper_1210_0461_b200.engine import worker_payloads  # noqa: F401

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_hash_coefficients_and_seeds_match_reference(golden):
    for case in golden["hashes"]:
        h = crop.make_hashes(crop.HashConfig(case["kappa"], case["seed"]))
        assert list(h.coefficients()) == case["coeffs"]
        assert h.row_hash.values(case["indices"]) == case["h_row"]
        assert h.col_hash.values(case["indices"]) == case["h_col"]
        for i, j, s in case["signs"]:
            assert h.sign_hash(i, j) == s
        assert hashing.hasher_to_text(h, case["seed"]) == case["text"]
        assert hashing.hasher_from_text(case["text"]) == h
    for m, lab, want in golden["derive_seed"]:
        assert crop.derive_seed(m, lab) == want
    for s, t, want in golden["instance_seeds"]:
        assert crop.EngineConfig(kappa=8, ss_capacity=4, seed=s, instances=t).instance_seeds() == want


def test_bucket_sort_indices_matches_reference(golden):
    for case in golden["bucket_sort"]:
        rm, ra = case["coeffs"][:2]
        v = crop.SparseVector(500, case["indices"], case["values"])
        out = crop.bucket_sort_indices(v, crop.IndexHashFn(rm, ra, case["kappa"]), case["combined"])
        assert out.hashes == case["hashes"]
        assert out.indices == case["sorted_indices"]
        assert out.values == case["sorted_values"]


def test_spacesaving_host_object_matches_reference(golden):
    for case in golden["spacesaving"]:
        s = crop.SpaceSavingSummary(case["capacity"])
        for item, w in case["updates"]:
            s.update(item, w)
        assert sorted([it, c, o] for it, c, o in s.records()) == sorted(case["records"])
        assert s.total_weight == case["total"]
        assert s.min_count() == case["min"]
        for q, want in case["queries"].items():
            assert list(s.query(q)) == want
    s = crop.SpaceSavingSummary(3)
    for (i, j), w in [((0, 1), 2.0), ((0, 2), 1.0), ((1, 2), 5.0)]:
        s.update((i, j), w)
    t = crop.SpaceSavingSummary.from_lines(s.to_lines())
    assert sorted(t.records()) == sorted(s.records())
    with pytest.raises(crop.InputError):
        s.update((0, 1), 0.0)


def test_config_and_assignment_validation():
    with pytest.raises(crop.ConfigError):
        crop.EngineConfig(kappa=0, ss_capacity=1)
    with pytest.raises(crop.ConfigError):
        crop.EngineConfig(kappa=4, ss_capacity=1, workers=5)
    with pytest.raises(crop.ConfigError):
        crop.EngineConfig(kappa=4, ss_capacity=1, instances=2)
    asg = crop.WorkerAssignment.split(10, 3)
    assert [(a.start, a.stop) for a in asg] == [(0, 3), (3, 6), (6, 10)]
    with pytest.raises(crop.ConfigError):
        crop.WorkerAssignment.split(3, 4)
    cfg = crop.EngineConfig(kappa=8, ss_capacity=4, workers=2)
    assert crop.EngineConfig.from_dict(cfg.to_dict()) == cfg


def test_sparse_types_and_streams(tmp_path):
    with pytest.raises(crop.InputError):
        crop.SparseVector(5, [2, 1], [1.0, 1.0])
    with pytest.raises(crop.DimensionError):
        crop.SparseVector(2, [0, 2], [1.0, 1.0])
    with pytest.raises(crop.InputError):
        crop.SparseVector(5, [1], [0.0])
    tx = [(0, 3, 5), (), (1,), (2, 3)]
    s = crop.transactions_to_stream(tx)
    assert s.n_rows == 6 and len(s) == 4
    assert s.transactions() == [tuple(t) for t in tx]
    assert [a.indices for a, b in s] == [tuple(t) for t in tx]
    assert s.pair_terms(True) == 3 + 0 + 0 + 1
    with pytest.raises(crop.InputError):
        crop.transactions_to_stream([(0, 9)], dim=5)
    with pytest.raises(crop.InputError):
        crop.TransactionStream(10, np.array([0, 2]), np.array([3, 3]))
    path = tmp_path / "t.dat"
    path.write_text("3 1 3\n\n2 2\n7 -1\n" if False else "3 1 3\n\n2 2 9\n")
    assert crop.read_fimi(path) == [(1, 3), (2, 9)]
    bad = tmp_path / "b.dat"
    bad.write_text("1 2\nx 3\n")
    with pytest.raises(crop.ParseError) as ei:
        crop.read_fimi(bad)
    assert ei.value.line_no == 2
    out = tmp_path / "w.dat"
    crop.write_fimi(out, [(1, 2), (3,)])
    assert crop.read_fimi(out) == [(1, 2), (3,)]


def test_triple_files(tmp_path):
    a = [crop.SparseVector(4, [0, 2], [1.5, -2.0]), crop.SparseVector(4, [], [])]
    b = [crop.SparseVector(4, [1], [3.0]), crop.SparseVector(4, [3], [1.0])]
    crop.write_triple_file(tmp_path / "a.txt", a, 4, 4)
    crop.write_triple_file(tmp_path / "b.txt", b, 4, 4)
    s = crop.load_column_row_streams(tmp_path / "a.txt", tmp_path / "b.txt")
    assert [(x.indices, x.values, y.indices, y.values) for x, y in s] == \
        [((0, 2), (1.5, -2.0), (1,), (3.0,)), ((), (), (3,), (1.0,))]
    (tmp_path / "c.txt").write_text("4 4 1\n0 1 zz\n")
    with pytest.raises(crop.ParseError):
        crop.load_column_row_streams(tmp_path / "c.txt", tmp_path / "b.txt")


def test_load_balance_and_report_logic():
    rep = crop.LoadReport(kappa=8, workers=4, rows=[[10, 10, 10, 10], [5, 15, 10, 10]],
                          input_pair_total=40)
    assert rep.total_entries == 40 and rep.expected_per_worker == 10
    assert rep.max_avg_ratio() == 1.5
    chk = crop.load_balance_check(rep, 0.2)
    assert (chk.violations, chk.checked) == (1, 2)
    rep.per_product = [(10, 10, [25, 25, 25, 25]), (1, 1, [1, 0, 0, 0])]
    chk = crop.load_balance_check(rep, 1.0)
    assert chk.checked == 1 and chk.violations == 0 and chk.bound == 1.0 / 20
    with pytest.raises(crop.ConfigError):
        crop.load_balance_check(rep, 0.0)


def _payload(cfg, worker, start, stop, count, summaries, hashes="h"):
    return {"format": "crop-partial/1", "worker": worker, "start": start, "stop": stop,
            "n_rows": 5, "n_cols": 5, "upper_triangle_only": True, "config": cfg.to_dict(),
            "instances": [{"seed": 1, "hashes": hashes, "count": count, "summaries": summaries,
                           "cs_cells": None}]}


def test_merge_partials_validation():
    cfg = crop.EngineConfig(kappa=4, ss_capacity=10, workers=2, cs_enabled=False)
    h = crop.make_hashes(crop.HashConfig(4, 1))
    text = hashing.hasher_to_text(h, 1)
    lines = ["capacity 10", "total_weight 3.0", "0 1 3.0 0.0"]
    p0 = _payload(cfg, 0, 0, 2, 3, [[1, lines]], text)
    p1 = _payload(cfg, 1, 2, 4, 0, [], text)
    state, rep = crop.merge_partials([p1, p0])
    assert rep.rows == [[3, 0]] and rep.input_pair_total == 0
    assert state.instances[0].summaries[1].query((0, 1)) == (3.0, 3.0)
    with pytest.raises(crop.InputError):
        crop.merge_partials([p0])
    with pytest.raises(crop.InputError):
        crop.merge_partials([p0, _payload(cfg, 1, 3, 4, 0, [], text)])
    with pytest.raises(crop.InputError):
        crop.merge_partials([p0, _payload(cfg, 1, 2, 4, 0, [[1, lines]], text)])
    with pytest.raises(crop.InputError):
        crop.merge_partials([])


def test_native_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "crop_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|const char\*|unsigned long long)\s+(crop_\w+)\(",
                              header, re.M))
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.EXPORTED)
    assert _native.load().crop_abi_version() == _native.ABI_VERSION


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(crop.DeviceError):
        crop.run(crop.transactions_to_stream([(0, 1)]), crop.EngineConfig(kappa=2, ss_capacity=4))


def test_workload_tables():
    th, al = workloads.zipf_alias(1000, 1.1)
    assert th.shape == al.shape == (1000,)
    # reconstruct the sampling probabilities from the alias table
    p = th.astype(np.float64) / 2 ** 32
    prob = p / 1000
    np.add.at(prob, al, (1 - p) / 1000)
    want = 1.0 / np.arange(1, 1001) ** 1.1
    want /= want.sum()
    np.testing.assert_allclose(prob, want, rtol=1e-6, atol=1e-9)
    cdf, lo = workloads.length_cdf(("poisson", 20, 2, 200))
    assert lo == 2 and cdf.shape == (199,) and cdf[-1] == 0xFFFFFFFF
    assert np.all(np.diff(cdf.astype(np.int64)) >= 0)
    cdf, lo = workloads.length_cdf(("uniform", 50, 300))
    assert cdf.shape == (251,)
    s = workloads.generate_product_workload(workloads.CONFIGS["c4"], n_products=2000)
    lens = np.diff(s.a_ptr)
    assert lens.min() >= 4 and lens.max() <= 2000
    for k in range(0, 2000, 97):
        seg = s.a_idx[s.a_ptr[k]:s.a_ptr[k + 1]]
        assert np.all(np.diff(seg.astype(np.int64)) > 0)


# ---------------------------------------------------------------- round 2

def test_max_avg_ratio_rounds_like_reference(golden):
    """engine.py:207-216: avg = total / len first, then max / avg, bit for bit."""
    for rows, want in golden["max_avg_ratio"]:
        rep = crop.LoadReport(kappa=len(rows[0]), workers=len(rows[0]), rows=rows,
                              input_pair_total=0)
        assert rep.max_avg_ratio() == want


def test_public_names_match_reference():
    ref_all = {"BalanceCheck", "ConfigError", "CountSketch", "CropError", "DimensionError",
               "EngineConfig", "Entry", "EntryHasher", "HashConfig", "HashedIndexArray",
               "IndexHashFn", "InputError", "LoadReport", "MedianEstimator",
               "OuterProductStream", "ParseError", "ResourceCapError", "ScanStats", "SignHashFn",
               "SketchState", "SpaceSavingSummary", "SparseVector", "TopEntry",
               "WorkerAssignment", "ZipfModel", "bound_ratio_report", "bucket_sort_indices",
               "count_interval", "derive_seed", "entry_hash", "enumerate_interval",
               "exact_pair_supports", "exact_product", "exact_top", "gen_zipf_stream",
               "gen_zipf_transactions", "load_balance_check", "load_column_row_streams",
               "load_state", "make_hashes", "measure_loads", "median_query", "merge_partials",
               "mine", "outer_product_nnz", "read_fimi", "recall_at_k", "run", "run_parallel",
               "run_worker", "save_state", "transaction_to_outer", "transactions_to_stream",
               "write_fimi", "write_triple_file"}  # reference __init__.py:84-137
    assert ref_all <= set(crop.__all__)
    assert all(hasattr(crop, n) for n in crop.__all__)


def test_zipf_generators_match_reference(golden):
    for case in golden["zipf"]["streams"]:
        scale, skew, distinct, dim, outer, seed = case["args"]
        s = crop.gen_zipf_stream(crop.ZipfModel(scale, skew, distinct), dim, outer, seed)
        got = [[list(a.indices), list(a.values), list(b.indices), list(b.values)] for a, b in s]
        assert got == case["products"]
    for case in golden["zipf"]["transactions"]:
        got = crop.gen_zipf_transactions(*case["args"])
        assert [list(t) for t in got] == case["transactions"]
    with pytest.raises(crop.ConfigError):
        crop.ZipfModel(0.0, 1.0, 3)
    with pytest.raises(crop.ConfigError):
        crop.gen_zipf_stream(crop.ZipfModel(1.0, 1.0, 50), 5, None, 0)
    with pytest.raises(crop.ConfigError):
        crop.gen_zipf_transactions(10, 5, 0.0, 0)


def test_cli_exit_codes_match_reference(golden, tmp_path):
    """cli.py:391-404 exit codes: a missing input is 2, a bad config is 3
    (both raised before any device work)."""
    from paper_1210_0461_b200 import cli

    codes = golden["cli"]["exit_codes"]
    fimi = tmp_path / "t.fimi"
    fimi.write_text(golden["cli"]["generate_transactions"]["fimi"])
    assert cli.main(["mine", "--fimi", str(tmp_path / "missing.fimi"), "--kappa", "4",
                     "--out", str(tmp_path / "x")]) == codes["missing_input"]
    assert cli.main(["mine", "--fimi", str(fimi), "--kappa", "4", "--workers", "9",
                     "--out", str(tmp_path / "y")]) == codes["bad_workers"]
    assert cli.main(["bench", "--kappa", "4", "--out", str(tmp_path / "z")]) == 2  # no input
    assert not (tmp_path / "x").exists() and not (tmp_path / "y").exists()
