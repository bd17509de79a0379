"""Sparse vectors, outer-product streams and their GPU-ready columnar forms.

API-compatible with the reference's `sparse.py` (`Entry` :16-20,
`SparseVector` :23-92, `OuterProductStream` :100-149, triple files
:152-264, FIMI :270-305). The B200 build adds two columnar stream types that
carry the whole stream as CSR arrays, which is what the kernels consume:

* `TransactionStream` -- a self-join stream (pair mining): transaction k is
  the 0/1 vector on both sides of product k (mining.py:15-22). Arrays:
  offsets int64[n+1], items uint32[nnz], ascending per transaction.
* `ColumnRowStream` -- a general stream a_k x b_k (A's columns as CSC, B's
  rows as CSR) with float64 values.

Both still iterate as (SparseVector, SparseVector) pairs, so any code written
against the reference keeps working; the engine recognises them and skips
the Python objects entirely.
"""

import logging
import os
from typing import Callable, Iterable, Iterator, NamedTuple

import numpy as np

from .errors import CropError, DimensionError, InputError, ParseError

logger = logging.getLogger(__name__)


class Entry(NamedTuple):
    row: int
    col: int


class SparseVector:
    """Immutable sparse vector: strictly increasing indices, non-zero values."""

    __slots__ = ("dim", "indices", "values")

    def __init__(self, dim: int, indices: Iterable[int], values: Iterable[float]):
        idx = tuple(int(i) for i in indices)
        val = tuple(float(v) for v in values)
        if dim < 0:
            raise DimensionError(f"negative dimension {dim}")
        if len(idx) != len(val):
            raise InputError(f"{len(idx)} indices but {len(val)} values")
        for a, b in zip(idx, idx[1:]):
            if b <= a:
                raise InputError(f"indices not strictly increasing at {b}")
        if idx and idx[0] < 0:
            raise InputError(f"indices not strictly increasing at {idx[0]}")
        if idx and idx[-1] >= dim:
            raise DimensionError(f"index {idx[-1]} out of range for dim {dim}")
        if any(v == 0.0 for v in val):
            raise InputError("stored values must be nonzero")
        object.__setattr__(self, "dim", dim)
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "values", val)

    def __setattr__(self, name, value):
        raise AttributeError("SparseVector is immutable")

    @classmethod
    def from_pairs(cls, dim: int, pairs: Iterable[tuple[int, float]]) -> "SparseVector":
        ordered = sorted(pairs)
        return cls(dim, [i for i, _ in ordered], [v for _, v in ordered])

    @property
    def nnz(self) -> int:
        return len(self.indices)

    def pairs(self) -> Iterator[tuple[int, float]]:
        return zip(self.indices, self.values)

    def get(self, index: int) -> float:
        pos = np.searchsorted(self.indices, index) if self.indices else 0
        if pos < len(self.indices) and self.indices[pos] == index:
            return self.values[pos]
        return 0.0

    def __reduce__(self):
        return (SparseVector, (self.dim, self.indices, self.values))

    def __eq__(self, other):
        return (isinstance(other, SparseVector) and self.dim == other.dim
                and self.indices == other.indices and self.values == other.values)

    def __hash__(self):
        return hash((self.dim, self.indices, self.values))

    def __repr__(self):
        return f"SparseVector(dim={self.dim}, nnz={self.nnz})"


def outer_product_nnz(a: SparseVector, b: SparseVector) -> int:
    return a.nnz * b.nnz


class OuterProductStream:
    """Re-iterable sequence of (column vector, row vector) pairs."""

    __slots__ = ("n_rows", "n_cols", "length", "_factory", "zero_values_dropped")

    def __init__(self, n_rows: int, n_cols: int, length: int,
                 factory: Callable[[], Iterable[tuple[SparseVector, SparseVector]]]):
        self.n_rows = n_rows
        self.n_cols = n_cols
        self.length = length
        self._factory = factory
        self.zero_values_dropped = 0

    @classmethod
    def from_pairs(cls, n_rows: int, n_cols: int,
                   pairs: Iterable[tuple[SparseVector, SparseVector]]) -> "OuterProductStream":
        pairs = list(pairs)
        for a, b in pairs:
            if a.dim != n_rows:
                raise DimensionError(f"left vector dim {a.dim} != n_rows {n_rows}")
            if b.dim != n_cols:
                raise DimensionError(f"right vector dim {b.dim} != n_cols {n_cols}")
        return cls(n_rows, n_cols, len(pairs), lambda: iter(pairs))

    def __iter__(self):
        return iter(self._factory())

    def __len__(self) -> int:
        return self.length

    def total_pair_count(self) -> int:
        return sum(a.nnz * b.nnz for a, b in self)

    def __repr__(self):
        return f"OuterProductStream({self.n_rows}x{self.n_cols}, {self.length} outer products)"


def _csr_from_lists(rows) -> tuple[np.ndarray, np.ndarray]:
    lens = np.fromiter((len(r) for r in rows), dtype=np.int64, count=len(rows))
    offsets = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    items = np.fromiter((i for r in rows for i in r), dtype=np.int64, count=int(offsets[-1]))
    return offsets, items


class TransactionStream(OuterProductStream):
    """Self-join stream over transactions stored as CSR (pair mining input):
    offsets int64[n + 1], items uint32[nnz] (or uint16 when passed as uint16
    and dim <= 65,536), strictly increasing within a transaction."""

    __slots__ = ("offsets", "items")

    def __init__(self, dim: int, offsets: np.ndarray, items: np.ndarray, validate: bool = True):
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        items_i64 = np.asarray(items)
        if validate:
            if offsets.ndim != 1 or offsets.shape[0] < 1 or offsets[0] != 0:
                raise InputError("offsets must be a 1-D array starting at 0")
            if np.any(np.diff(offsets) < 0) or offsets[-1] != items_i64.shape[0]:
                raise InputError("offsets must be non-decreasing and end at len(items)")
            if items_i64.size:
                if items_i64.min() < 0:
                    raise InputError(f"negative item id {int(items_i64.min())}")
                if items_i64.max() >= dim:
                    raise InputError(f"item id {int(items_i64.max())} outside configured "
                                     f"universe [0, {dim})")
                d = np.diff(items_i64.astype(np.int64))
                inner = np.ones(d.shape[0], dtype=bool)  # d[x] compares items x, x+1
                cuts = offsets[1:-1]
                inner[cuts[(cuts > 0) & (cuts < items_i64.shape[0])] - 1] = False
                if np.any(inner & (d <= 0)):
                    raise InputError("items must be strictly increasing within a transaction")
        self.offsets = offsets
        # ids stay uint16 when given so (half the bytes to move to the device)
        keep16 = items_i64.dtype == np.uint16 and dim <= 65536
        self.items = np.ascontiguousarray(items_i64, dtype=np.uint16 if keep16 else np.uint32)
        n = offsets.shape[0] - 1
        super().__init__(dim, dim, n, self._pairs)

    def _pairs(self):
        off, it = self.offsets, self.items
        for k in range(self.length):
            v = SparseVector(self.n_rows, it[off[k]:off[k + 1]].tolist(),
                             [1.0] * int(off[k + 1] - off[k]))
            yield v, v

    @classmethod
    def from_transactions(cls, transactions, dim: int | None = None) -> "TransactionStream":
        rows = [tuple(t) for t in transactions]
        offsets, items = _csr_from_lists(rows)
        max_item = int(items.max()) if items.size else -1
        if dim is None:
            dim = max_item + 1
        elif max_item >= dim:
            raise InputError(f"item id {max_item} outside configured universe [0, {dim})")
        return cls(dim, offsets, items)

    @property
    def nnz(self) -> int:
        return int(self.offsets[-1])

    def pair_terms(self, upper_only: bool = True) -> int:
        lens = np.diff(self.offsets)
        return int((lens * (lens - 1) // 2).sum()) if upper_only else int((lens * lens).sum())

    def total_pair_count(self) -> int:
        lens = np.diff(self.offsets)
        return int((lens * lens).sum())

    def transactions(self) -> list[tuple[int, ...]]:
        off, it = self.offsets, self.items
        return [tuple(it[off[k]:off[k + 1]].tolist()) for k in range(self.length)]


class ColumnRowStream(OuterProductStream):
    """General stream: a_k = A[:, k] (CSC) and b_k = B[k, :] (CSR), float64 values."""

    __slots__ = ("a_ptr", "a_idx", "a_val", "b_ptr", "b_idx", "b_val")

    def __init__(self, n_rows, n_cols, a_ptr, a_idx, a_val, b_ptr, b_idx, b_val):
        self.a_ptr = np.ascontiguousarray(a_ptr, dtype=np.int64)
        self.a_idx = np.ascontiguousarray(a_idx, dtype=np.uint32)
        self.a_val = np.ascontiguousarray(a_val, dtype=np.float64)
        self.b_ptr = np.ascontiguousarray(b_ptr, dtype=np.int64)
        self.b_idx = np.ascontiguousarray(b_idx, dtype=np.uint32)
        self.b_val = np.ascontiguousarray(b_val, dtype=np.float64)
        if self.a_ptr.shape != self.b_ptr.shape:
            raise DimensionError(f"k-count mismatch: {self.a_ptr.shape[0] - 1} columns vs "
                                 f"{self.b_ptr.shape[0] - 1} rows")
        super().__init__(n_rows, n_cols, self.a_ptr.shape[0] - 1, self._pairs)

    def _pairs(self):
        for k in range(self.length):
            a0, a1 = self.a_ptr[k], self.a_ptr[k + 1]
            b0, b1 = self.b_ptr[k], self.b_ptr[k + 1]
            yield (SparseVector(self.n_rows, self.a_idx[a0:a1].tolist(), self.a_val[a0:a1].tolist()),
                   SparseVector(self.n_cols, self.b_idx[b0:b1].tolist(), self.b_val[b0:b1].tolist()))

    @classmethod
    def from_stream(cls, stream: OuterProductStream) -> "ColumnRowStream":
        if isinstance(stream, ColumnRowStream):
            return stream
        if isinstance(stream, TransactionStream):
            v = np.ones(stream.items.shape[0])
            return cls(stream.n_rows, stream.n_cols, stream.offsets, stream.items, v,
                       stream.offsets, stream.items, v)
        a_rows, a_vals, b_rows, b_vals = [], [], [], []
        for a, b in stream:
            a_rows.append(a.indices)
            a_vals.append(a.values)
            b_rows.append(b.indices)
            b_vals.append(b.values)
        a_ptr, a_idx = _csr_from_lists(a_rows)
        b_ptr, b_idx = _csr_from_lists(b_rows)
        a_val = np.fromiter((v for r in a_vals for v in r), dtype=np.float64, count=a_idx.shape[0])
        b_val = np.fromiter((v for r in b_vals for v in r), dtype=np.float64, count=b_idx.shape[0])
        out = cls(stream.n_rows, stream.n_cols, a_ptr, a_idx, a_val, b_ptr, b_idx, b_val)
        out.zero_values_dropped = stream.zero_values_dropped
        return out

    def total_pair_count(self) -> int:
        return int((np.diff(self.a_ptr) * np.diff(self.b_ptr)).sum())

    def is_binary_self_join(self) -> bool:
        return (np.array_equal(self.a_ptr, self.b_ptr) and np.array_equal(self.a_idx, self.b_idx)
                and bool(np.all(self.a_val == 1.0)) and bool(np.all(self.b_val == 1.0))
                and self.n_rows == self.n_cols)


def as_transaction_stream(stream: OuterProductStream) -> TransactionStream | None:
    """The self-join 0/1 view of a stream, or None when it is not one."""
    if isinstance(stream, TransactionStream):
        return stream
    if stream.n_rows != stream.n_cols:
        return None
    if isinstance(stream, ColumnRowStream):
        return (TransactionStream(stream.n_rows, stream.a_ptr, stream.a_idx, validate=False)
                if stream.is_binary_self_join() else None)
    rows = []
    for a, b in stream:
        if a is not b and (a.indices != b.indices or a.values != b.values):
            return None
        if any(v != 1.0 for v in a.values):
            return None
        rows.append(a.indices)
    offsets, items = _csr_from_lists(rows)
    return TransactionStream(stream.n_rows, offsets, items, validate=False)


# --- triple files (sparse.py:152-264) --------------------------------------

def _read_header(path, line: str, line_no: int) -> tuple[int, int, int]:
    parts = line.split()
    if len(parts) != 3:
        raise ParseError(path, line_no, f"expected 'n_rows n_cols kcount', got {line!r}")
    try:
        n_rows, n_cols, kcount = (int(p) for p in parts)
    except ValueError:
        raise ParseError(path, line_no, f"non-integer header field in {line!r}") from None
    if min(n_rows, n_cols, kcount) < 0:
        raise ParseError(path, line_no, "header fields must be nonnegative")
    return n_rows, n_cols, kcount


def read_triple_file(path):
    """Parse one side's triple file -> (n_rows, n_cols, groups, zeros dropped)."""
    try:
        with open(path, "r", encoding="utf-8") as fh:
            lines = fh.read().splitlines()
    except OSError as exc:
        raise InputError(f"cannot read {path}: {exc}") from exc
    if not lines:
        raise ParseError(path, 1, "missing header line")
    n_rows, n_cols, kcount = _read_header(path, lines[0], 1)
    groups: list[list[tuple[int, float]]] = [[] for _ in range(kcount)]
    zeros = 0
    last_k = -1
    for line_no, line in enumerate(lines[1:], start=2):
        parts = line.split()
        if not parts:
            continue
        if len(parts) != 3:
            raise ParseError(path, line_no, f"expected 'k index value', got {line!r}")
        try:
            k, idx, val = int(parts[0]), int(parts[1]), float(parts[2])
        except ValueError:
            raise ParseError(path, line_no, f"malformed triple {line!r}") from None
        if k < last_k:
            raise ParseError(path, line_no, f"k values not sorted: {k} after {last_k}")
        last_k = k
        if not 0 <= k < kcount:
            raise ParseError(path, line_no, f"k={k} outside [0, {kcount})")
        if idx < 0:
            raise ParseError(path, line_no, f"negative index {idx}")
        if val != val:
            raise ParseError(path, line_no, "NaN value")
        if val == 0.0:
            zeros += 1
            continue
        groups[k].append((idx, val))
    for k, g in enumerate(groups):
        g.sort()
        for (i1, _), (i2, _) in zip(g, g[1:]):
            if i1 == i2:
                raise ParseError(path, 0, f"duplicate index {i1} within k={k}")
    if zeros:
        logger.warning("%s: dropped %d explicit-zero triples", path, zeros)
    return n_rows, n_cols, groups, zeros


def read_triple_csr(path, threads: int = 0):
    """read_triple_file into CSR over k: (n_rows, n_cols, ptr int64[kcount+1],
    idx uint32, val float64, zeros dropped), parsed by the native
    multi-threaded reader (csrc/ingest.cu). Files it does not accept -- every
    error and every unusual spelling -- are re-read by the reference-exact
    read_triple_file, which raises the reference's ParseError / InputError."""
    import ctypes

    from . import _native as nat

    try:
        lib = nat.load()
    except CropError:
        lib = None
    if lib is not None:
        h = ctypes.c_void_p()
        dims = (ctypes.c_int64 * 3)()
        nnz, zeros, bad = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        rc = lib.crop_triple_parse(os.fsencode(str(path)), int(threads), ctypes.byref(h), dims,
                                   ctypes.byref(nnz), ctypes.byref(zeros), ctypes.byref(bad))
        if rc == 0:
            try:
                ptr = _host_array(dims[2] + 1, np.int64)
                idx = _host_array(nnz.value, np.uint32)
                val = np.empty(nnz.value, dtype=np.float64)
                nat.check(lib.crop_triple_copy(h, ptr.ctypes.data, idx.ctypes.data, val.ctypes.data))
            finally:
                lib.crop_triple_free(h)
            if zeros.value:
                logger.warning("%s: dropped %d explicit-zero triples", path, zeros.value)
            return int(dims[0]), int(dims[1]), ptr, idx, val, int(zeros.value)
    n_rows, n_cols, groups, z = read_triple_file(path)
    ptr, idx = _csr_from_lists([[i for i, _ in g] for g in groups])
    val = np.array([v for g in groups for _, v in g], dtype=np.float64)
    return n_rows, n_cols, ptr, idx.astype(np.uint32), val, z


def load_column_row_streams(path_a, path_b) -> ColumnRowStream:
    """Load A's columns and B's rows (sparse.py:228-254) as one columnar
    stream, both files parsed by the native reader."""
    ar, ac, a_ptr, a_idx, a_val, za = read_triple_csr(path_a)
    br, bc, b_ptr, b_idx, b_val, zb = read_triple_csr(path_b)
    if a_ptr.shape[0] != b_ptr.shape[0]:
        raise DimensionError(f"k-count mismatch: {path_a} has {a_ptr.shape[0] - 1}, "
                             f"{path_b} has {b_ptr.shape[0] - 1}")
    if (ar, ac) != (br, bc):
        raise DimensionError(f"header mismatch: {path_a} says {ar}x{ac}, {path_b} says {br}x{bc}")
    for ptr, idx, dim in ((a_ptr, a_idx, ar), (b_ptr, b_idx, bc)):
        if idx.size and int(idx.max()) >= dim:
            k = int(np.searchsorted(ptr, int(np.argmax(idx >= dim)), side="right")) - 1
            last = int(idx[ptr[k]:ptr[k + 1]].max())
            raise DimensionError(f"k={k}: index {last} out of range for dim {dim}")
    s = ColumnRowStream(ar, bc, a_ptr, a_idx, a_val, b_ptr, b_idx, b_val)
    s.zero_values_dropped = za + zb
    return s


def _load_column_row_streams_lists(path_a, path_b) -> ColumnRowStream:
    ar, ac, ga, za = read_triple_file(path_a)
    br, bc, gb, zb = read_triple_file(path_b)
    if len(ga) != len(gb):
        raise DimensionError(f"k-count mismatch: {path_a} has {len(ga)}, {path_b} has {len(gb)}")
    if (ar, ac) != (br, bc):
        raise DimensionError(f"header mismatch: {path_a} says {ar}x{ac}, {path_b} says {br}x{bc}")
    for k, (x, y) in enumerate(zip(ga, gb)):
        if x and x[-1][0] >= ar:
            raise DimensionError(f"k={k}: index {x[-1][0]} out of range for dim {ar}")
        if y and y[-1][0] >= bc:
            raise DimensionError(f"k={k}: index {y[-1][0]} out of range for dim {bc}")
    a_ptr, a_idx = _csr_from_lists([[i for i, _ in g] for g in ga])
    b_ptr, b_idx = _csr_from_lists([[i for i, _ in g] for g in gb])
    a_val = np.array([v for g in ga for _, v in g], dtype=np.float64)
    b_val = np.array([v for g in gb for _, v in g], dtype=np.float64)
    s = ColumnRowStream(ar, bc, a_ptr, a_idx, a_val, b_ptr, b_idx, b_val)
    s.zero_values_dropped = za + zb
    return s


def write_triple_file(path, vectors: Iterable[SparseVector], n_rows: int, n_cols: int) -> None:
    vectors = list(vectors)
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"{n_rows} {n_cols} {len(vectors)}\n")
        for k, vec in enumerate(vectors):
            for idx, val in vec.pairs():
                fh.write(f"{k} {idx} {val!r}\n")


# --- FIMI transaction files (sparse.py:270-305) -----------------------------

def read_fimi(path) -> list[tuple[int, ...]]:
    """One transaction per line of integer ids; deduplicated and sorted."""
    out = []
    dups = 0
    try:
        with open(path, "r", encoding="utf-8") as fh:
            for line_no, line in enumerate(fh, start=1):
                parts = line.split()
                if not parts:
                    continue
                try:
                    ids = [int(p) for p in parts]
                except ValueError:
                    raise ParseError(path, line_no,
                                     f"non-integer item in {line.strip()!r}") from None
                if min(ids) < 0:
                    raise ParseError(path, line_no, f"negative item id {min(ids)}")
                uniq = tuple(sorted(set(ids)))
                dups += len(ids) - len(uniq)
                out.append(uniq)
    except OSError as exc:
        raise InputError(f"cannot read {path}: {exc}") from exc
    if dups:
        logger.warning("%s: dropped %d duplicate items within transactions", path, dups)
    return out


def _host_array(n: int, dtype) -> np.ndarray:
    """A numpy array in pinned (page-locked) memory when a GPU is present, so
    the one host -> device copy of the stream runs at full DMA speed."""
    try:
        import torch

        if torch.cuda.is_available():
            tdt = {np.int64: torch.int64, np.uint32: torch.int32}[dtype]
            return torch.empty(max(n, 1), dtype=tdt, pin_memory=True).numpy().view(dtype)[:n]
    except Exception:
        pass
    return np.empty(n, dtype=dtype)


def read_fimi_csr(path, threads: int = 0) -> tuple[np.ndarray, np.ndarray, int]:
    """read_fimi into CSR (offsets int64, items uint32, max id or -1) with the
    native multi-threaded reader; lines the native reader does not accept
    (errors or unusual forms) are handed to the reference-exact read_fimi,
    which raises the same ParseError / InputError as the reference."""
    import ctypes

    from . import _native as nat

    lib = nat.load()
    h = ctypes.c_void_p()
    n_tx, nnz, dups, bad = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    mx = ctypes.c_uint32()
    rc = lib.crop_fimi_parse(os.fsencode(str(path)), int(threads), ctypes.byref(h), ctypes.byref(n_tx),
                             ctypes.byref(nnz), ctypes.byref(mx), ctypes.byref(dups), ctypes.byref(bad))
    if rc != 0:
        rows = read_fimi(path)
        offsets, items = _csr_from_lists(rows)
        return offsets, items.astype(np.uint32), (int(items.max()) if items.size else -1)
    try:
        offsets = _host_array(n_tx.value + 1, np.int64)
        items = _host_array(nnz.value, np.uint32)
        nat.check(lib.crop_fimi_copy(h, offsets.ctypes.data, items.ctypes.data))
    finally:
        lib.crop_fimi_free(h)
    if dups.value:
        logger.warning("%s: dropped %d duplicate items within transactions", path, dups.value)
    return offsets, items, (int(mx.value) if nnz.value else -1)


def write_fimi(path, transactions: Iterable[Iterable[int]]) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for items in transactions:
            fh.write(" ".join(str(i) for i in items) + "\n")
