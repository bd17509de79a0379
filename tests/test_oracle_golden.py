"""Pin the C oracle (oracle/crop_oracle.c) to the reference's own outputs.

The fixtures in tests/golden/reference_golden.json were produced by running
the reference package (tests/golden/make_golden.py). If these pass, the
oracle restates the reference bit for bit on integer work and sums real
weights in the reference's order.
"""

import numpy as np
import pytest

import oracle
from conftest import tx_to_csr, vectors_to_csr


def test_index_and_sign_hash(golden):
    for case in golden["hashes"]:
        rm, ra, cm, ca, sm, sa = case["coeffs"]
        got_r = oracle.index_hash(case["indices"], rm, ra, case["kappa"])
        got_c = oracle.index_hash(case["indices"], cm, ca, case["kappa"])
        assert got_r.tolist() == case["h_row"]
        assert got_c.tolist() == case["h_col"]
        for i, j, s in case["signs"]:
            assert oracle.sign_hash(i, j, sm, sa) == s


def test_mulmod61_against_python_ints():
    rng = np.random.default_rng(0)
    p = oracle.MERSENNE_PRIME
    for _ in range(2000):
        a = int(rng.integers(1, p))
        b = int(rng.integers(0, 2 ** 63)) * 2 + int(rng.integers(0, 2))
        c = int(rng.integers(0, p))
        assert oracle.mulmod61(a, b, c) == (a * b + c) % p


def test_bucket_sort(golden):
    for case in golden["bucket_sort"]:
        rm, ra = case["coeffs"][:2]
        h = oracle.index_hash(case["indices"], rm, ra, case["kappa"])
        comb = -1 if case["combined"] is None else case["combined"]
        oh, oi, ov = oracle.bucket_sort(case["indices"], case["values"], h, case["kappa"], comb)
        assert oh.tolist() == case["hashes"]
        assert oi.tolist() == case["sorted_indices"]
        assert ov.tolist() == case["sorted_values"]


def _records_by_bucket(recs):
    return sorted((int(b), int(r), int(c), float(n), float(o)) for b, r, c, n, o in recs)


@pytest.mark.parametrize("case_idx", range(5))
def test_mining_run_matches_reference(golden, case_idx):
    case = golden["mining"][case_idx]
    cfg = case["config"]
    off, items = tx_to_csr(case["transactions"])
    stream = oracle.Stream(off, items)
    exact = cfg["ss_capacity"] >= 2 ** 31
    for k, inst in enumerate(case["instances"]):
        recs, loads = oracle.run(stream, inst["coeffs"], cfg["kappa"], cfg["workers"],
                                 capacity=0 if exact else cfg["ss_capacity"], upper_only=True,
                                 cs=True)
        got = _records_by_bucket(zip(recs.bucket, recs.row, recs.col, recs.count, recs.over))
        want = _records_by_bucket(inst["records"])
        assert got == want
        assert loads.tolist() == case["rows"][k]
        assert recs.cs.tolist() == inst["cs"]
        for b, tot in inst["bucket_totals"].items():
            assert recs.bucket_totals[int(b)] == tot
        ml, total = oracle.measure_loads(stream, inst["coeffs"], cfg["kappa"], cfg["workers"], True)
        assert ml.tolist() == case["loads_upper"][k]
        ml, total = oracle.measure_loads(stream, inst["coeffs"], cfg["kappa"], cfg["workers"], False)
        assert ml.tolist() == case["loads_full"][k]
        assert total == case["pair_total_full"]


@pytest.mark.parametrize("case_idx", range(5))
def test_parallel_and_worker_runs_are_k_invariant(golden, case_idx):
    case = golden["mining"][case_idx]
    cfg = case["config"]
    off, items = tx_to_csr(case["transactions"])
    stream = oracle.Stream(off, items)
    exact = cfg["ss_capacity"] >= 2 ** 31
    inst = case["instances"][0]
    cap = 0 if exact else cfg["ss_capacity"]
    recs, loads = oracle.run_parallel(stream, inst["coeffs"], cfg["kappa"], cfg["workers"],
                                      capacity=cap, upper_only=True, threads=3)
    got = _records_by_bucket(zip(recs.bucket, recs.row, recs.col, recs.count, recs.over))
    assert got == _records_by_bucket(inst["records"])
    assert loads.tolist() == case["rows"][0]
    for w in range(cfg["workers"]):
        r, load = oracle.run_worker(stream, inst["coeffs"], cfg["kappa"], cfg["workers"], w,
                                    capacity=cap, upper_only=True)
        assert load == case["rows"][0][w]


def test_pair_supports(golden):
    for case in golden["mining"]:
        off, items = tx_to_csr(case["transactions"])
        r, c, w = oracle.sorted_pairs(*oracle.pair_supports(off, items))
        got = [[int(a), int(b), int(x)] for a, b, x in zip(r, c, w)]
        assert got == case["supports"]


def test_selfjoin_full(golden):
    case = golden["selfjoin_full"]
    cfg = case["config"]
    off, items = tx_to_csr(case["transactions"])
    inst = case["instances"][0]
    recs, loads = oracle.run(oracle.Stream(off, items), inst["coeffs"], cfg["kappa"],
                             cfg["workers"], upper_only=False, cs=True)
    got = _records_by_bucket(zip(recs.bucket, recs.row, recs.col, recs.count, recs.over))
    assert got == _records_by_bucket(inst["records"])
    assert loads.tolist() == case["rows"][0]
    assert recs.cs.tolist() == inst["cs"]


def test_general_products(golden):
    for case in golden["general"]:
        ap, ai, av = vectors_to_csr(case["a"])
        bp, bi, bv = vectors_to_csr(case["b"])
        s = oracle.Stream(ap, ai, av, bp, bi, bv)
        r, c, w = oracle.sorted_pairs(*oracle.exact_product(s))
        assert [[int(a), int(b), float(x)] for a, b, x in zip(r, c, w)] == case["exact"]
        r, c, w = oracle.sorted_pairs(*oracle.exact_product(s, upper_only=True))
        assert [[int(a), int(b), float(x)] for a, b, x in zip(r, c, w)] == case["exact_upper"]
        for w_idx, part in enumerate(case["partitions"]):
            recs, load = oracle.run_worker(s, case["coeffs"], case["kappa"], case["workers"],
                                           w_idx)
            got = sorted([int(a), int(b), float(x)] for a, b, x in
                         zip(recs.row, recs.col, recs.count))
            assert got == part["entries"]
            assert load == part["count"]
