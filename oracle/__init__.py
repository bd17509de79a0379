"""CPU oracle for the CRoP hot path -- TEST INFRASTRUCTURE ONLY.

This package is the checker, never the product. Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it; `paper_1210_0461_b200` never does (its kernels fail
loudly when the CUDA library is missing instead of falling back here).

It wraps `oracle/crop_oracle.c` (a plain-C restatement of the reference
functions, each citing its reference file:line) through ctypes. The
restatement is pinned to the Python reference by tests/golden/*.json, which
tests/golden/make_golden.py produced by importing the reference itself.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libcrop_oracle.so")
_lib = None

MERSENNE_PRIME = (1 << 61) - 1


def build(force: bool = False) -> str:
    """Compile the oracle library with the committed Makefile."""
    src = os.path.join(_HERE, "crop_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, u64, u32, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        L.ora_mulmod61.restype = u64
        L.ora_mulmod61.argtypes = [u64, u64, u64]
        L.ora_index_hash.argtypes = [P, i64, u64, u64, u32, P]
        L.ora_sign_hash.restype = i32
        L.ora_sign_hash.argtypes = [u32, u32, u64, u64]
        L.ora_bucket_sort.argtypes = [P, P, i64, P, u32, i64, P, P, P]
        L.ora_run.restype = P
        L.ora_run.argtypes = [P, P, P, P, P, P, i64, P, u32, i32, i64, i32, i32, P]
        L.ora_run_worker.restype = P
        L.ora_run_worker.argtypes = [P, P, P, P, P, P, i64, P, u32, i32, i32, i64, i32, i32, P]
        L.ora_run_parallel.restype = P
        L.ora_run_parallel.argtypes = [P, P, P, P, P, P, i64, P, u32, i32, i64, i32, i32, i32, P]
        L.ora_measure_loads.argtypes = [P, P, P, P, i64, P, u32, i32, i32, P, P]
        L.ora_result_size.restype = i64
        L.ora_result_size.argtypes = [P]
        L.ora_result_export.argtypes = [P, P, P, P, P, P]
        L.ora_result_loads.argtypes = [P, P]
        L.ora_result_cs.restype = i32
        L.ora_result_cs.argtypes = [P, P]
        L.ora_result_bucket_totals.argtypes = [P, P]
        L.ora_result_free.argtypes = [P]
        L.ora_pair_supports.restype = P
        L.ora_pair_supports.argtypes = [P, P, i64]
        L.ora_exact_product.restype = P
        L.ora_exact_product.argtypes = [P, P, P, P, P, P, i64, i32]
        L.ora_table_size.restype = i64
        L.ora_table_size.argtypes = [P]
        L.ora_table_export.argtypes = [P, P, P, P]
        L.ora_table_free.argtypes = [P]
        L.ora_gen_lengths.argtypes = [i64, u64, P, u32, u32, P]
        L.ora_gen_lengths.restype = None
        L.ora_gen_items.argtypes = [i64, u64, u32, P, P, P, P, i32]
        L.ora_gen_items.restype = None
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _coeffs(coeffs):
    return np.ascontiguousarray([int(c) for c in coeffs], dtype=np.uint64)


# ---------------------------------------------------------------- hashing

def mulmod61(a: int, b: int, c: int) -> int:
    return int(lib().ora_mulmod61(a, b, c))


def index_hash(indices, mul: int, add: int, kappa: int) -> np.ndarray:
    idx = _u32(indices)
    out = np.empty(idx.shape[0], dtype=np.uint32)
    lib().ora_index_hash(_p(idx), idx.shape[0], mul, add, kappa, _p(out))
    return out


def sign_hash(row: int, col: int, mul: int, add: int) -> int:
    return int(lib().ora_sign_hash(row, col, mul, add))


def bucket_sort(indices, values, hashes, kappa: int, combined: int = -1):
    idx, h = _u32(indices), _u32(hashes)
    val = _f64(values)
    n = idx.shape[0]
    oh, oi, ov = np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.float64)
    lib().ora_bucket_sort(_p(idx), _p(val), n, _p(h), kappa, combined, _p(oh), _p(oi), _p(ov))
    return oh, oi, ov


# ---------------------------------------------------------------- results

class Records:
    """Per-bucket records exported from an oracle run (numpy columns)."""

    def __init__(self, handle, kappa: int, cs: bool):
        L = lib()
        n = int(L.ora_result_size(handle))
        self.bucket = np.empty(n, np.uint32)
        self.row = np.empty(n, np.uint32)
        self.col = np.empty(n, np.uint32)
        self.count = np.empty(n, np.float64)
        self.over = np.empty(n, np.float64)
        L.ora_result_export(handle, _p(self.bucket), _p(self.row), _p(self.col), _p(self.count),
                            _p(self.over))
        self.bucket_loads = np.empty(kappa, np.uint64)
        L.ora_result_loads(handle, _p(self.bucket_loads))
        self.bucket_totals = np.empty(kappa, np.float64)
        L.ora_result_bucket_totals(handle, _p(self.bucket_totals))
        self.cs = None
        if cs:
            self.cs = np.empty(kappa, np.float64)
            L.ora_result_cs(handle, _p(self.cs))
        L.ora_result_free(handle)

    def as_dict(self) -> dict:
        return {(int(r), int(c)): float(w) for r, c, w in zip(self.row, self.col, self.count)}


class Stream:
    """Compressed outer-product stream: left/right CSR arrays (self-join when
    the right side is omitted)."""

    def __init__(self, a_ptr, a_idx, a_val=None, b_ptr=None, b_idx=None, b_val=None):
        self.a_ptr, self.a_idx, self.a_val = _i64(a_ptr), _u32(a_idx), _f64(a_val)
        if b_ptr is None:
            self.b_ptr, self.b_idx, self.b_val = self.a_ptr, self.a_idx, self.a_val
        else:
            self.b_ptr, self.b_idx, self.b_val = _i64(b_ptr), _u32(b_idx), _f64(b_val)
        self.n = self.a_ptr.shape[0] - 1

    def args(self):
        return (_p(self.a_ptr), _p(self.a_idx), _p(self.a_val), _p(self.b_ptr), _p(self.b_idx),
                _p(self.b_val), self.n)


def run(stream: Stream, coeffs, kappa: int, workers: int, capacity: int = 0,
        upper_only: bool = False, cs: bool = False):
    """engine.run for one instance (capacity <= 0: exact regime)."""
    loads = np.zeros(workers, np.uint64)
    h = lib().ora_run(*stream.args(), _p(_coeffs(coeffs)), kappa, workers, capacity,
                      int(upper_only), int(cs), _p(loads))
    return Records(h, kappa, cs), loads


def run_worker(stream: Stream, coeffs, kappa: int, workers: int, worker: int,
               capacity: int = 0, upper_only: bool = False, cs: bool = False):
    load = np.zeros(1, np.uint64)
    h = lib().ora_run_worker(*stream.args(), _p(_coeffs(coeffs)), kappa, workers, worker,
                             capacity, int(upper_only), int(cs), _p(load))
    return Records(h, kappa, cs), int(load[0])


def run_parallel(stream: Stream, coeffs, kappa: int, workers: int, capacity: int = 0,
                 upper_only: bool = False, cs: bool = False, threads: int = 1):
    loads = np.zeros(workers, np.uint64)
    h = lib().ora_run_parallel(*stream.args(), _p(_coeffs(coeffs)), kappa, workers, capacity,
                               int(upper_only), int(cs), threads, _p(loads))
    return Records(h, kappa, cs), loads


def measure_loads(stream: Stream, coeffs, kappa: int, workers: int, upper_only: bool = False):
    loads = np.zeros(workers, np.uint64)
    total = np.zeros(1, np.uint64)
    lib().ora_measure_loads(_p(stream.a_ptr), _p(stream.a_idx), _p(stream.b_ptr),
                            _p(stream.b_idx), stream.n, _p(_coeffs(coeffs)), kappa, workers,
                            int(upper_only), _p(loads), _p(total))
    return loads, int(total[0])


def _table(handle):
    L = lib()
    n = int(L.ora_table_size(handle))
    row, col, w = np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.float64)
    L.ora_table_export(handle, _p(row), _p(col), _p(w))
    L.ora_table_free(handle)
    return row, col, w


def pair_supports(offsets, items):
    """exact_pair_supports (oracle.py:61-71) -> (row, col, support) arrays."""
    off, it = _i64(offsets), _u32(items)
    return _table(lib().ora_pair_supports(_p(off), _p(it), off.shape[0] - 1))


def exact_product(stream: Stream, upper_only: bool = False):
    """exact_product (oracle.py:20-50) -> (row, col, weight), zero sums dropped."""
    row, col, w = _table(lib().ora_exact_product(*stream.args(), int(upper_only)))
    keep = w != 0.0
    return row[keep], col[keep], w[keep]


def sorted_pairs(row, col, w):
    """Canonical (row, col)-sorted view for comparisons."""
    order = np.lexsort((col, row))
    return row[order], col[order], w[order]


def gen_transactions(n_tx: int, n_items: int, item_alias, len_cdf, len_lo: int, seed: int,
                     threads: int = 0):
    """Host copy of the bench's seeded generator (csrc/gen.cu, restated in
    crop_oracle.c) -> CSR (offsets int64[n_tx+1], items uint32[nnz]); the same
    arrays the GPU generator writes, without loading the product library."""
    thresh, alias = _u32(item_alias[0]), _u32(item_alias[1])
    cdf = _u32(len_cdf)
    lengths = np.empty(max(n_tx, 1), np.int64)
    lib().ora_gen_lengths(n_tx, seed, _p(cdf), cdf.shape[0], len_lo, _p(lengths))
    offsets = np.zeros(n_tx + 1, np.int64)
    np.cumsum(lengths[:n_tx], out=offsets[1:])
    items = np.empty(max(int(offsets[-1]), 1), np.uint32)
    threads = threads or len(os.sched_getaffinity(0))
    lib().ora_gen_items(n_tx, seed, n_items, _p(thresh), _p(alias), _p(offsets), _p(items),
                        threads)
    return offsets, items[: int(offsets[-1])]
