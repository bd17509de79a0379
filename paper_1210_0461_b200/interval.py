"""Interval-restricted enumeration of outer-product entries (drop-in for interval.py).

The reference's Lemma-1 scan (`interval.py:125-189`) walks one outer product
with four monotone cursors over hash-sorted index arrays. On the GPU the
same selection -- entries (i, j) with (h_row(i) + h_col(j)) mod kappa in
[start, stop) -- is evaluated for a whole batch of products at once
(csrc/outer.cu, csrc/crop_api.cu); the per-product helpers here keep the
reference's signatures and results:

* `WorkerAssignment.split` (:20-45) and `bucket_sort_indices` (:70-109) are
  host utilities (bucket_sort_indices reproduces the (hash, index) order of
  both reference branches);
* `enumerate_interval` (:236-254) and `count_interval` (:257-269) run on the
  device and return the reference's emission order (left position, right
  position in hash-sorted order, :134-138).
"""

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError
from .hashing import IndexHashFn
from .sparse import Entry, SparseVector


@dataclass(frozen=True)
class WorkerAssignment:
    """Half-open bucket interval [start, stop) of [0, kappa) owned by one worker."""

    start: int
    stop: int
    kappa: int

    def __post_init__(self):
        if not 0 <= self.start <= self.stop <= self.kappa:
            raise ConfigError(f"invalid interval [{self.start}, {self.stop}) for kappa={self.kappa}")

    def __len__(self) -> int:
        return self.stop - self.start

    @classmethod
    def split(cls, kappa: int, workers: int) -> list["WorkerAssignment"]:
        if not 1 <= workers <= kappa:
            raise ConfigError(f"workers must be in [1, kappa], got {workers} for kappa={kappa}")
        cuts = [c * kappa // workers for c in range(workers + 1)]
        return [cls(cuts[c], cuts[c + 1], kappa) for c in range(workers)]


class HashedIndexArray:
    """A vector's indices sorted by (hash, index), values riding along."""

    __slots__ = ("hashes", "indices", "values")

    def __init__(self, hashes, indices, values):
        self.hashes = hashes
        self.indices = indices
        self.values = values

    def __len__(self) -> int:
        return len(self.hashes)

    def pairs(self):
        return list(zip(self.hashes, self.indices))


def bucket_sort_indices(v: SparseVector, index_hash: IndexHashFn,
                        combined_nnz: int | None = None) -> HashedIndexArray:
    """Stable sort of v's indices by hash value (both reference branches agree)."""
    if v.nnz == 0:
        return HashedIndexArray([], [], [])
    h = index_hash.values(v.indices)
    order = np.argsort(np.asarray(h, dtype=np.int64), kind="stable")  # indices ascending already
    return HashedIndexArray([h[p] for p in order], [v.indices[p] for p in order],
                            [v.values[p] for p in order])


@dataclass
class ScanStats:
    """Operation counts. For the GPU path: `element_checks` counts the
    (i, j) candidates the kernel evaluated, `emitted` the entries produced."""

    cursor_moves: int = 0
    element_checks: int = 0
    emitted: int = 0
    products: int = 0

    def total_ops(self) -> int:
        return self.cursor_moves + self.element_checks + self.emitted


def _check_kappa(row_hash: IndexHashFn, col_hash: IndexHashFn, assignment: WorkerAssignment):
    if not (row_hash.kappa == col_hash.kappa == assignment.kappa):
        raise ConfigError(f"kappa mismatch: row {row_hash.kappa}, col {col_hash.kappa}, "
                          f"interval {assignment.kappa}")


def _single_product(a: SparseVector, b: SparseVector):
    from .sparse import ColumnRowStream

    return ColumnRowStream(max(a.dim, 1), max(b.dim, 1),
                           np.array([0, a.nnz]), np.array(a.indices, dtype=np.uint32),
                           np.array(a.values), np.array([0, b.nnz]),
                           np.array(b.indices, dtype=np.uint32), np.array(b.values))


def _tables(row_hash: IndexHashFn, col_hash: IndexHashFn, n_items: int):
    from . import kernels
    from .hashing import EntryHasher, SignHashFn

    h = EntryHasher(row_hash, col_hash, SignHashFn(1, 0, row_hash.prime))
    return kernels.hash_tables(h, n_items)


def enumerate_interval(a: SparseVector, b: SparseVector, row_hash: IndexHashFn,
                       col_hash: IndexHashFn, assignment: WorkerAssignment,
                       stats: ScanStats | None = None):
    """Yield (Entry, a(i)*b(j)) for the entries of a*b whose bucket is in the interval."""
    from . import kernels

    _check_kappa(row_hash, col_hash, assignment)
    if stats is not None:
        stats.products += 1
        stats.element_checks += a.nnz * b.nnz
    if a.nnz == 0 or b.nnz == 0 or assignment.start == assignment.stop:
        return
    n_items = 1 + max(max(a.indices), max(b.indices))
    h_row, h_col = _tables(row_hash, col_hash, n_items)
    ds = kernels.DeviceOuterStream.from_host(_single_product(a, b))
    ent = kernels.outer_product(ds, False, row_hash.kappa, assignment.start, assignment.stop,
                                h_row, h_col)
    rows, cols, vals = ent.to_numpy()
    # reference emission order: left then right position in (hash, index) order
    ra = np.asarray(row_hash.values(rows.tolist()), dtype=np.int64)
    cb = np.asarray(col_hash.values(cols.tolist()), dtype=np.int64)
    order = np.lexsort((cols, cb, rows, ra))
    if stats is not None:
        stats.emitted += int(order.shape[0])
    for p in order:
        yield Entry(int(rows[p]), int(cols[p])), float(vals[p])


def count_interval(a: SparseVector, b: SparseVector, row_hash: IndexHashFn,
                   col_hash: IndexHashFn, assignment: WorkerAssignment) -> int:
    """Number of entries enumerate_interval would yield (device bucket-load kernel)."""
    from . import kernels

    _check_kappa(row_hash, col_hash, assignment)
    if a.nnz == 0 or b.nnz == 0 or assignment.start == assignment.stop:
        return 0
    n_items = 1 + max(max(a.indices), max(b.indices))
    h_row, h_col = _tables(row_hash, col_hash, n_items)
    ds = kernels.DeviceOuterStream.from_host(_single_product(a, b))
    loads = kernels.outer_bucket_loads(ds, h_row, h_col, row_hash.kappa, False)
    return int(loads[assignment.start:assignment.stop].sum().item())
