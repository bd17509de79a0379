"""Thin torch-facing wrappers over the C-ABI (one function per kernel family).

Device buffers are torch CUDA tensors (uint32 data is carried in int32
tensors, uint64 in int64); every call is ordered on the current CUDA stream.
Nothing here falls back to the CPU: without the library or a device the
calls raise `DeviceError` (see `_native.require_cuda`).
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .errors import ConfigError, DeviceError, InputError, ResourceCapError

TOPK_EXACT_BINS = 2048       # topk histogram: exact below, 2^-10 relative above
TOPK_BINS = 2048 + 21 * 1024  # common.cuh kTopkBins
U32_MASK = 0xFFFFFFFF


def _dev():
    return nat.require_cuda()


def u32_to_numpy(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


# ------------------------------------------------------------------ inputs

@dataclass
class DeviceTransactions:
    """Transactions resident in HBM: CSR offsets int64[n+1], items uint32[nnz]."""

    offsets: torch.Tensor
    items: torch.Tensor
    n_items: int

    @property
    def n_tx(self) -> int:
        return self.offsets.shape[0] - 1

    @property
    def n_rows(self) -> int:
        return self.n_items

    n_cols = n_rows

    @property
    def nnz(self) -> int:
        return self.items.shape[0]

    @classmethod
    def from_host(cls, offsets: np.ndarray, items: np.ndarray, n_items: int,
                  non_blocking: bool = False) -> "DeviceTransactions":
        dev = _dev()
        off = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64))
        items = np.asarray(items)
        if items.dtype == np.uint16:
            # 16-bit ids travel as they are and widen on the device
            it = torch.from_numpy(np.ascontiguousarray(items).view(np.int16))
        else:
            it = torch.from_numpy(np.ascontiguousarray(items, dtype=np.uint32).view(np.int32))
        if non_blocking:
            off, it = off.pin_memory(), it.pin_memory()
        it = it.to(dev, non_blocking=non_blocking)
        if it.dtype == torch.int16:
            it = it.to(torch.int32) & 0xFFFF
        return cls(off.to(dev, non_blocking=non_blocking), it, int(n_items))

    def to_host(self) -> tuple[np.ndarray, np.ndarray]:
        return self.offsets.cpu().numpy(), u32_to_numpy(self.items)

    def slice(self, t0: int, t1: int, host_offsets: np.ndarray | None = None) -> "DeviceTransactions":
        """Transactions [t0, t1) as their own stream (item ids shared, offsets
        rebased); host_offsets (the host copy of offsets) avoids a read-back."""
        if host_offsets is not None:
            i0, i1 = int(host_offsets[t0]), int(host_offsets[t1])
        else:
            i0, i1 = (int(x) for x in self.offsets[[t0, t1]].tolist())
        items = self.items[i0:i1]
        if i0 % 4:
            items = items.clone()  # the counting kernels read 16-byte aligned item vectors
        return DeviceTransactions(self.offsets[t0:t1 + 1] - i0, items, self.n_items)


@dataclass
class DeviceOuterStream:
    """General stream in HBM: a_k (CSC column) x b_k (CSR row), float64 values."""

    a_ptr: torch.Tensor
    a_idx: torch.Tensor
    a_val: torch.Tensor
    b_ptr: torch.Tensor
    b_idx: torch.Tensor
    b_val: torch.Tensor
    n_rows: int
    n_cols: int

    @property
    def n_products(self) -> int:
        return self.a_ptr.shape[0] - 1

    def shape(self) -> "nat.OuterShape":
        """All terms, largest row / column index and nonzero counts, reduced on
        the device once per stream (one read-back) and cached: every job over
        this stream then plans without synchronising."""
        cached = getattr(self, "_shape", None)
        if cached is None:
            n = self.n_products
            if n > 0 and self.a_idx.numel() and self.b_idx.numel():
                la = self.a_ptr[1:] - self.a_ptr[:-1]
                lb = self.b_ptr[1:] - self.b_ptr[:-1]
                mask = 0xFFFFFFFF
                vals = torch.stack([(la * lb).sum(), self.a_idx.to(torch.int64).bitwise_and(mask).max(),
                                    self.b_idx.to(torch.int64).bitwise_and(mask).max()]).tolist()
            else:
                vals = [0, 0, 0]
            cached = nat.OuterShape(int(vals[0]), int(vals[1]), int(vals[2]), int(self.a_idx.numel()),
                                    int(self.b_idx.numel()))
            object.__setattr__(self, "_shape", cached)
        return cached

    @classmethod
    def from_host(cls, s, non_blocking: bool = False) -> "DeviceOuterStream":
        dev = _dev()

        def up(a, dt, view=None):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=dt) if view is None else
                                 np.ascontiguousarray(a, dtype=dt).view(view))
            if non_blocking:
                t = t.pin_memory()
            return t.to(dev, non_blocking=non_blocking)

        return cls(up(s.a_ptr, np.int64), up(s.a_idx, np.uint32, np.int32), up(s.a_val, np.float64),
                   up(s.b_ptr, np.int64), up(s.b_idx, np.uint32, np.int32), up(s.b_val, np.float64),
                   s.n_rows, s.n_cols)


# ------------------------------------------------------------------ hashing

def hash_tables(hasher, n_items: int) -> tuple[torch.Tensor, torch.Tensor]:
    """K0: (h_row, h_col) uint32[n_items] for one EntryHasher (hashing.py:68-71)."""
    dev = _dev()
    kappa = hasher.kappa
    if kappa > (1 << 31):
        raise ConfigError(f"kappa {kappa} exceeds the device limit 2^31")
    n = max(int(n_items), 1)
    h_row = torch.empty(n, dtype=torch.int32, device=dev)
    h_col = torch.empty(n, dtype=torch.int32, device=dev)
    nat.call("crop_hash_tables", int(n_items), hasher.row_hash.mul, hasher.row_hash.add,
             hasher.col_hash.mul, hasher.col_hash.add, kappa, nat.ptr(h_row), nat.ptr(h_col),
             nat.stream_ptr())
    return h_row, h_col


def sign_hash(row: torch.Tensor, col: torch.Tensor, sign_fn) -> torch.Tensor:
    out = torch.empty(row.shape[0], dtype=torch.int8, device=row.device)
    nat.call("crop_sign_hash", nat.ptr(row), nat.ptr(col), row.shape[0], sign_fn.mul, sign_fn.add,
             nat.ptr(out), nat.stream_ptr())
    return out


def interval_struct(kappa: int, start: int, stop: int, h_row=None, h_col=None) -> nat.Interval:
    return nat.Interval(kappa, start, stop, nat.ptr(h_row), nat.ptr(h_col))


# ------------------------------------------------------------------ K1 loads

def selfjoin_bucket_loads(dtx: DeviceTransactions, h_row, h_col, kappa: int,
                          upper_only: bool) -> torch.Tensor:
    loads = torch.zeros(kappa, dtype=torch.int64, device=dtx.offsets.device)
    nat.call("crop_selfjoin_bucket_loads", nat.ptr(dtx.offsets), nat.ptr(dtx.items), dtx.n_tx,
             nat.ptr(h_row), nat.ptr(h_col), kappa, int(upper_only), nat.ptr(loads),
             nat.stream_ptr())
    return loads


def outer_bucket_loads(ds: DeviceOuterStream, h_row, h_col, kappa: int,
                       upper_only: bool) -> torch.Tensor:
    loads = torch.zeros(kappa, dtype=torch.int64, device=ds.a_ptr.device)
    nat.call("crop_outer_bucket_loads", nat.ptr(ds.a_ptr), nat.ptr(ds.a_idx), nat.ptr(ds.b_ptr),
             nat.ptr(ds.b_idx), ds.n_products, nat.ptr(h_row), nat.ptr(h_col), kappa,
             int(upper_only), nat.ptr(loads), nat.stream_ptr())
    return loads


# ------------------------------------------------------------------ K2 pairs

@dataclass
class DeviceEntries:
    """Counted entries in HBM (unordered): row, col uint32 and a weight column.

    `count` (uint32) for 0/1 streams, `value` (float64) for real streams;
    `bucket` is filled by the real-valued path (sorted per bucket)."""

    row: torch.Tensor
    col: torch.Tensor
    count: torch.Tensor | None
    value: torch.Tensor | None
    n: int
    total_terms: int
    bucket: torch.Tensor | None = None
    # fused top-k inputs filled by the counting kernels (stream-mode jobs):
    # (hist int32[23552], hi_list int64[], hi_n int64[1])
    topk_fused: tuple | None = None

    def weights_f64(self) -> torch.Tensor:
        if self.value is not None:
            return self.value[: self.n]
        return (self.count[: self.n].to(torch.int64) & U32_MASK).to(torch.float64)

    def weights_at(self, idx: torch.Tensor) -> torch.Tensor:
        """float64 weights of the entries `idx` (gather first, convert after)."""
        if self.value is not None:
            return self.value[idx]
        return (self.count[idx].to(torch.int64) & U32_MASK).to(torch.float64)

    def to_numpy(self):
        row = u32_to_numpy(self.row[: self.n])
        col = u32_to_numpy(self.col[: self.n])
        w = self.weights_f64().cpu().numpy()
        return row, col, w


class PairCountJob:
    """K2 handle: plan on create (one stream sync), run on demand."""

    def __init__(self, dtx: DeviceTransactions, upper_only: bool, interval: nat.Interval | None,
                 keep: tuple = (), shard: tuple[int, int] = (0, 1), flags: int = 0):
        """shard = (rank, world): keep this rank's share of the tiles (the union
        over ranks is the whole job; crop_pairs_create_sharded). flags:
        CROP_PAIRS_* of crop_pairs_create_ex."""
        self._keep = (dtx, keep)  # tensors the native job points at
        self.dtx = dtx
        self._args = (upper_only, interval, keep, shard, flags)
        lib = nat.load()
        h = ctypes.c_void_p()
        iv = ctypes.byref(interval) if interval is not None else None
        nat.check(lib.crop_pairs_create_ex(nat.ptr(dtx.offsets), nat.ptr(dtx.items), dtx.n_tx,
                                           dtx.n_items, int(upper_only), iv, int(shard[0]),
                                           int(shard[1]), int(flags), nat.stream_ptr(),
                                           ctypes.byref(h)))
        self._h = h
        own = ctypes.c_int()
        nat.check(lib.crop_pairs_own(h, ctypes.byref(own)))
        self.own = bool(own.value)
        me, tt, nt, nu = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        nat.check(lib.crop_pairs_info(h, ctypes.byref(me), ctypes.byref(tt), ctypes.byref(nt),
                                      ctypes.byref(nu)))
        self.max_entries, self.total_terms = int(me.value), int(tt.value)
        self.n_tiles, self.n_units = int(nt.value), int(nu.value)
        ot = ctypes.c_uint64()
        nat.check(lib.crop_pairs_own_terms(h, ctypes.byref(ot)))
        self.own_terms = int(ot.value)  # 0: unknown
        self.sharded = shard[1] > 1

    def run(self, sync: bool = True, capacity: int | None = None) -> DeviceEntries:
        """Count; output arrays hold `capacity` entries (default: a guess of half
        the terms, bounded by max_entries). With sync, an output that did not
        fit is counted again with the full bound."""
        dev = self.dtx.offsets.device
        if capacity is None:
            if self.sharded and self.own_terms:
                # a shard emits at most one entry per own term (c3's light
                # shards are almost all distinct pairs)
                capacity = min(self.max_entries, self.own_terms + (1 << 20))
            else:
                capacity = min(self.max_entries, self.total_terms // 2 + (1 << 20))
        m = max(min(int(capacity), self.max_entries), 1)
        nat.check(nat.load().crop_pairs_set_capacity(self._h, m))
        row = torch.empty(m, dtype=torch.int32, device=dev)
        col = torch.empty(m, dtype=torch.int32, device=dev)
        cnt = torch.empty(m, dtype=torch.int32, device=dev)
        n_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        fused = None
        if self.stream_mode:
            hi_cap = self.total_terms // TOPK_EXACT_BINS + 1
            hist = torch.zeros(TOPK_BINS, dtype=torch.int32, device=dev)
            hi_n = torch.zeros(1, dtype=torch.int64, device=dev)
            hi_list = torch.empty(hi_cap, dtype=torch.int64, device=dev)
            nat.check(nat.load().crop_pairs_set_topk(self._h, nat.ptr(hist), nat.ptr(hi_list),
                                                     nat.ptr(hi_n), hi_cap))
            fused = (hist, hi_list, hi_n)
        nat.check(nat.load().crop_pairs_run(self._h, nat.ptr(row), nat.ptr(col), nat.ptr(cnt),
                                            nat.ptr(n_dev), nat.stream_ptr()))
        if fused is not None:
            nat.check(nat.load().crop_pairs_set_topk(self._h, None, None, None, 0))
        ent = DeviceEntries(row, col, cnt, None, -1, self.total_terms, topk_fused=fused)
        ent.n_dev = n_dev
        ent.capacity = m
        if sync:
            ent.n = int(n_dev.item())
            if ent.n > m:
                if m >= self.max_entries:
                    raise InputError(f"pair engine overflow: {ent.n} > {self.max_entries}")
                # the counter claims every entry even past the capacity: the
                # re-run needs exactly n slots
                n_need = ent.n
                del ent, row, col, cnt, fused
                return self.run(True, min(self.max_entries, n_need))
            if self.overflowed():
                upper_only, interval, keep, shard, flags = self._args
                if self.stream_mode and not flags & nat.PAIRS_SAFE_UNITS:
                    # a 16-bit counter wrapped (adversarial stream order):
                    # re-plan with units of <= 65,535 words and count again
                    del ent, row, col, cnt, fused
                    safe = PairCountJob(self.dtx, upper_only, interval, keep, shard,
                                        flags | nat.PAIRS_SAFE_UNITS)
                    try:
                        return safe.run(True, capacity)
                    finally:
                        safe.close()
                raise InputError("pair engine overflow: counts exceeded their bounds")
        return ent

    def set_timing(self, on: bool = True) -> None:
        nat.check(nat.load().crop_pairs_set_timing(self._h, int(on)))

    def phase_ms(self) -> dict:
        out = (ctypes.c_float * 4)()
        nat.check(nat.load().crop_pairs_phase_ms(self._h, out))
        return {"route": out[0], "write": out[1], "count": out[3]}

    @property
    def stream_mode(self) -> bool:
        """True when the job counts per-pair word streams (see crop_pairs_mode)."""
        flag = ctypes.c_int()
        nat.check(nat.load().crop_pairs_mode(self._h, ctypes.byref(flag)))
        return bool(flag.value)

    def overflowed(self) -> bool:
        flag = ctypes.c_int()
        nat.check(nat.load().crop_pairs_overflowed(self._h, ctypes.byref(flag)))
        return bool(flag.value)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            nat.load().crop_pairs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def count_pairs(dtx: DeviceTransactions, upper_only: bool = True, kappa: int = 1, start: int = 0,
                stop: int | None = None, h_row=None, h_col=None) -> DeviceEntries:
    """Exact supports of the entries whose bucket lies in [start, stop)."""
    stop = kappa if stop is None else stop
    iv = None
    if not (start == 0 and stop == kappa):
        if h_row is None or h_col is None:
            raise ConfigError("a partial interval needs the hash tables")
        iv = interval_struct(kappa, start, stop, h_row, h_col)
    return count_pairs_shard(dtx, upper_only, iv, (h_row, h_col), (0, 1))


def count_pairs_shard(dtx: DeviceTransactions, upper_only: bool, interval, keep=(),
                      shard: tuple[int, int] = (0, 1), capacity: int | None = None,
                      max_split: int = 64) -> DeviceEntries:
    """Exact supports of one tile shard; a shard whose entry lists exceed one
    job's 2^32 limit is counted as k consecutive sub-shards (r*k + s of N*k,
    s < k -- together exactly the tiles of a finer split's shards, so the
    union over all ranks is still the whole job, disjoint)."""
    r, world = shard
    k = 1
    while True:
        parts = []
        try:
            for s in range(k):
                job = PairCountJob(dtx, upper_only, interval, keep=keep, shard=(r * k + s, world * k))
                try:
                    parts.append(job.run(capacity=capacity))
                finally:
                    job.close()
        except ResourceCapError:
            if k >= max_split:
                raise
            del parts
            k *= 2
            continue
        break
    if len(parts) == 1:
        return parts[0]
    n = sum(p.n for p in parts)
    cat = lambda xs: torch.cat(xs) if xs else torch.empty(0, dtype=torch.int32, device=dtx.offsets.device)
    ent = DeviceEntries(cat([p.row[: p.n] for p in parts]), cat([p.col[: p.n] for p in parts]),
                        cat([p.count[: p.n] for p in parts]), None, n, parts[0].total_terms)
    ent.n_dev = torch.tensor([n], dtype=torch.int64, device=dtx.offsets.device)
    ent.capacity = n
    ent.sub_shards = k
    return ent


def entry_bucket_stats(ent: DeviceEntries, tables: list, kappa: int, n_items: int,
                       signs: list | None):
    """Per-instance (loads, distinct, cs) of counted entries; tables[t]=(h_row,h_col)."""
    dev = ent.row.device
    t = len(tables)
    h_row = torch.cat([x[0][:n_items] for x in tables]) if t > 1 else tables[0][0]
    h_col = torch.cat([x[1][:n_items] for x in tables]) if t > 1 else tables[0][1]
    loads = torch.zeros(t * kappa, dtype=torch.int64, device=dev)
    distinct = torch.zeros(t * kappa, dtype=torch.int32, device=dev)
    cs = torch.zeros(t * kappa, dtype=torch.int64, device=dev) if signs else None
    sg = None
    if signs:
        sg = (ctypes.c_uint64 * (2 * t))(*[v for s in signs for v in (s.mul, s.add)])
    n_dev = getattr(ent, "n_dev", None)
    if n_dev is None:
        n_dev = torch.tensor([ent.n], dtype=torch.int64, device=dev)
    nat.call("crop_entry_bucket_stats", nat.ptr(ent.row), nat.ptr(ent.col), nat.ptr(ent.count),
             nat.ptr(n_dev), ent.row.shape[0], t, n_items,
             nat.ptr(h_row), nat.ptr(h_col), kappa, sg, nat.ptr(loads), nat.ptr(distinct),
             nat.ptr(cs), nat.stream_ptr())
    return loads.view(t, kappa), distinct.view(t, kappa), (cs.view(t, kappa) if cs is not None else None)


def entry_buckets(row, col, n: int, h_row, h_col, kappa: int) -> torch.Tensor:
    out = torch.empty(max(n, 1), dtype=torch.int32, device=row.device)
    nat.call("crop_entry_buckets", nat.ptr(row), nat.ptr(col), n, nat.ptr(h_row), nat.ptr(h_col),
             kappa, nat.ptr(out), nat.stream_ptr())
    return out[:n]


# ------------------------------------------------------------------ K4 top-k

def launch_counter() -> int:
    return int(nat.load().crop_launch_counter())


def topk_indices(ent: DeviceEntries, k: int, count: torch.Tensor | None = None) -> torch.Tensor:
    """Indices of the best k entries by (count desc, row asc, col asc), unordered."""
    dev = ent.row.device
    cnt = ent.count if count is None else count
    k = int(k)
    out = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
    kout = torch.zeros(1, dtype=torch.int64, device=dev)
    n_dev = getattr(ent, "n_dev", None)
    if n_dev is None:
        n_dev = torch.tensor([ent.n], dtype=torch.int64, device=dev)
    if count is None and ent.topk_fused is not None:
        hist, hi_list, hi_n = ent.topk_fused
        nat.call("crop_topk_fused", nat.ptr(ent.row), nat.ptr(ent.col), nat.ptr(cnt), nat.ptr(n_dev),
                 ent.row.shape[0], k, nat.ptr(hist), nat.ptr(hi_list), nat.ptr(hi_n), nat.ptr(out),
                 nat.ptr(kout), nat.stream_ptr())
    else:
        nat.call("crop_topk", nat.ptr(ent.row), nat.ptr(ent.col), nat.ptr(cnt), nat.ptr(n_dev),
                 ent.row.shape[0], k, nat.ptr(out), nat.ptr(kout), nat.stream_ptr())
    return out[: int(kout.item())]


def bucket_topk(ent: DeviceEntries, h_row, h_col, kappa: int, capacity: int, want_mask: bool = True):
    """Per-bucket top-`capacity` of integer entries by (count desc, row, col):
    (recorded bool[n] or None, bucket_min int64[kappa], bucket_total int64[kappa])
    -- the bounded Space-Saving summaries (csrc/bucket_topk.cu)."""
    dev = ent.row.device
    n_dev = getattr(ent, "n_dev", None)
    if n_dev is None:
        n_dev = torch.tensor([ent.n], dtype=torch.int64, device=dev)
    cap = min(int(capacity), 0xFFFFFFFF)
    rec = torch.empty(max(ent.n, 1), dtype=torch.uint8, device=dev) if want_mask else None
    bmin = torch.empty(kappa, dtype=torch.int32, device=dev)
    btot = torch.empty(kappa, dtype=torch.int32, device=dev)
    nat.call("crop_bucket_topk", nat.ptr(ent.row), nat.ptr(ent.col), nat.ptr(ent.count), nat.ptr(n_dev),
             ent.row.shape[0], nat.ptr(h_row), nat.ptr(h_col), int(kappa), cap,
             nat.ptr(rec) if rec is not None else None, nat.ptr(bmin), nat.ptr(btot), nat.stream_ptr())
    mask = rec[: ent.n].to(torch.bool) if rec is not None else None
    return mask, bmin.to(torch.int64) & U32_MASK, btot.to(torch.int64) & U32_MASK


# ------------------------------------------------------------------ streaming Space-Saving

class StreamingSummaries:
    """Per-bucket Space-Saving summaries of one instance with O(l) device
    state (csrc/ss_stream.cu): flat records (row, col, count, over) of every
    bucket, at most `capacity` per bucket, and mu[b] = the minimum count of a
    full bucket (its upper bound for unrecorded keys). absorb() merges the
    exact entries of one chunk of the stream (spacesaving.py:39-63 applied to
    the chunk's aggregated weights; see the header of ss_stream.cu)."""

    def __init__(self, kappa: int, capacity: int, tables):
        dev = _dev()
        self.kappa, self.capacity = int(kappa), int(capacity)
        self.h_row, self.h_col = tables
        self.row = torch.empty(0, dtype=torch.int32, device=dev)
        self.col = torch.empty(0, dtype=torch.int32, device=dev)
        self.count = torch.empty(0, dtype=torch.int32, device=dev)
        self.over = torch.empty(0, dtype=torch.int32, device=dev)
        self.mu = torch.zeros(kappa, dtype=torch.int32, device=dev)
        self.per_bucket = torch.zeros(kappa, dtype=torch.int64, device=dev)

    @property
    def n(self) -> int:
        return int(self.row.shape[0])

    def state_bytes(self) -> int:
        """Device bytes of the summaries themselves (16 B per record)."""
        return 16 * self.n + 4 * self.kappa

    def absorb(self, ent: DeviceEntries) -> None:
        dev = self.mu.device
        n_rec, n_e = self.n, int(ent.n)
        if n_e == 0:
            return
        slots = 1024
        while slots < 2 * n_rec:
            slots <<= 1
        index = torch.empty(slots, dtype=torch.int64, device=dev)
        # Bloom filter over the record keys: at most 4 keys per 64-bit word up
        # to 2^23 words (64 MB; c3: 9 keys per word. Measured on a c3 chunk
        # merge: 2^21 75 ms, 2^22 77, 2^23 47, 2^24 50, 2^25 55); none for a
        # handful of records
        bloom_words = 0
        if n_rec >= 4096:
            bloom_words = 1024
            while bloom_words < n_rec // 4 and bloom_words < (1 << 23):
                bloom_words <<= 1
        bloom = torch.empty(bloom_words, dtype=torch.int64, device=dev) if bloom_words else None
        nat.call("crop_ss_index", nat.ptr(self.row), nat.ptr(self.col), n_rec, nat.ptr(index), slots,
                 nat.ptr(bloom), bloom_words, nat.stream_ptr())
        n_dev = getattr(ent, "n_dev", None)
        if n_dev is None:
            n_dev = torch.tensor([n_e], dtype=torch.int64, device=dev)
        # pass 1: hits add to their records; misses are flagged and counted per
        # bucket and chunk weight, which gives every bucket its cut
        missbits = torch.empty((n_e + 31) // 32, dtype=torch.int32, device=dev)
        hist = torch.empty(self.kappa * 16, dtype=torch.int32, device=dev)
        cut = torch.empty(self.kappa, dtype=torch.int32, device=dev)
        meta = torch.empty(2, dtype=torch.int64, device=dev)
        sat = torch.zeros(1, dtype=torch.int32, device=dev)
        nat.call("crop_ss_probe", nat.ptr(ent.row), nat.ptr(ent.col), nat.ptr(ent.count), nat.ptr(n_dev), n_e,
                 nat.ptr(index), slots, nat.ptr(bloom), bloom_words, n_rec,
                 nat.ptr(self.h_row), nat.ptr(self.h_col), self.kappa,
                 min(self.capacity, 0xFFFFFFFF), nat.ptr(self.row), nat.ptr(self.col), nat.ptr(self.count),
                 nat.ptr(missbits), nat.ptr(hist), nat.ptr(cut), nat.ptr(meta), nat.ptr(sat), nat.stream_ptr())
        del index, bloom
        n_cand = int(meta[0].item())
        # pass 2: the misses at or above their bucket's cut, behind the records
        m = n_rec + n_cand
        row = torch.empty(m, dtype=torch.int32, device=dev)
        col = torch.empty(m, dtype=torch.int32, device=dev)
        cnt = torch.empty(m, dtype=torch.int32, device=dev)
        over = torch.empty(m, dtype=torch.int32, device=dev)
        row[:n_rec], col[:n_rec], cnt[:n_rec], over[:n_rec] = self.row, self.col, self.count, self.over
        n_out = torch.tensor([n_rec], dtype=torch.int64, device=dev)
        nat.call("crop_ss_append", nat.ptr(ent.row), nat.ptr(ent.col), nat.ptr(ent.count), nat.ptr(n_dev), n_e,
                 nat.ptr(missbits), nat.ptr(cut), nat.ptr(meta), nat.ptr(self.h_row), nat.ptr(self.h_col),
                 self.kappa, nat.ptr(self.mu), nat.ptr(row), nat.ptr(col), nat.ptr(cnt), nat.ptr(over),
                 nat.ptr(n_out), nat.ptr(sat), nat.stream_ptr())
        del missbits
        n_tot, saturated = (int(x) for x in torch.cat([n_out, sat.to(torch.int64)]).tolist())
        if saturated:
            raise ResourceCapError("a Space-Saving count passed 2^32 - 1")
        if n_tot != m:
            raise DeviceError(f"summary merge: {n_tot - n_rec} candidates appended, {n_cand} counted")
        self.last_candidates = n_cand
        comb = DeviceEntries(row, col, cnt, None, n_tot, 0)
        comb.n_dev = n_out
        rec = torch.empty(max(n_tot, 1), dtype=torch.uint8, device=dev)
        bmin = torch.empty(self.kappa, dtype=torch.int32, device=dev)
        per = torch.empty(self.kappa, dtype=torch.int32, device=dev)
        nat.call("crop_bucket_topk", nat.ptr(row), nat.ptr(col), nat.ptr(cnt), nat.ptr(n_out), m,
                 nat.ptr(self.h_row), nat.ptr(self.h_col), self.kappa, min(self.capacity, 0xFFFFFFFF),
                 nat.ptr(rec), nat.ptr(bmin), nat.ptr(per), nat.stream_ptr())
        bmin = bmin.to(torch.int64) & U32_MASK
        per = per.to(torch.int64) & U32_MASK
        keep_n = int(torch.minimum(per, torch.full_like(per, self.capacity)).sum().item())
        out = [torch.empty(max(keep_n, 1), dtype=torch.int32, device=dev) for _ in range(4)]
        n_keep = torch.zeros(1, dtype=torch.int64, device=dev)
        nat.call("crop_ss_keep", nat.ptr(rec), nat.ptr(n_out), n_tot, nat.ptr(row), nat.ptr(col), nat.ptr(cnt),
                 nat.ptr(over), *[nat.ptr(o) for o in out], nat.ptr(n_keep), nat.stream_ptr())
        del rec, row, col, cnt, over
        self.row, self.col, self.count, self.over = (o[:keep_n] for o in out)
        full = per >= self.capacity
        self.per_bucket = torch.minimum(per, torch.full_like(per, self.capacity))
        self.mu = torch.where(full, bmin, torch.zeros_like(bmin)).to(torch.int32)


# ------------------------------------------------------------------ K5 outer

def outer_product(ds: DeviceOuterStream, upper_only: bool = False, kappa: int = 1, start: int = 0,
                  stop: int | None = None, h_row=None, h_col=None) -> DeviceEntries:
    """Per-bucket sorted COO of the stream restricted to buckets [start, stop)."""
    stop = kappa if stop is None else stop
    iv = interval_struct(kappa, start, stop, h_row, h_col) if h_row is not None else None
    if iv is None and not (start == 0 and stop == kappa):
        raise ConfigError("a partial interval needs the hash tables")
    lib = nat.load()
    h = ctypes.c_void_p()
    shape = ds.shape()
    nat.check(lib.crop_outer_create_ex(nat.ptr(ds.a_ptr), nat.ptr(ds.a_idx), nat.ptr(ds.a_val),
                                       nat.ptr(ds.b_ptr), nat.ptr(ds.b_idx), nat.ptr(ds.b_val),
                                       ds.n_products, int(upper_only),
                                       ctypes.byref(iv) if iv is not None else None,
                                       ctypes.byref(shape), nat.stream_ptr(), ctypes.byref(h)))
    try:
        me, tt = ctypes.c_uint64(), ctypes.c_uint64()
        nat.check(lib.crop_outer_info(h, ctypes.byref(me), ctypes.byref(tt)))
        m = max(int(me.value), 1)
        dev = ds.a_ptr.device
        row = torch.empty(m, dtype=torch.int32, device=dev)
        col = torch.empty(m, dtype=torch.int32, device=dev)
        val = torch.empty(m, dtype=torch.float64, device=dev)
        buck = torch.empty(m, dtype=torch.int32, device=dev)
        n_dev = torch.zeros(2, dtype=torch.int64, device=dev)
        nat.check(lib.crop_outer_run(h, nat.ptr(row), nat.ptr(col), nat.ptr(val), nat.ptr(buck),
                                     nat.ptr(n_dev), nat.stream_ptr()))
        nat.check(lib.crop_outer_own_terms(h, ctypes.c_void_p(n_dev.data_ptr() + 8), nat.stream_ptr()))
        n, own = n_dev.tolist()
    finally:
        lib.crop_outer_destroy(h)
    ent = DeviceEntries(row, col, None, val, n, own, bucket=buck)
    ent.n_dev = n_dev
    return ent


# ------------------------------------------------------------------ generator

def generate_transactions(n_tx: int, n_items: int, item_alias: tuple, len_cdf: np.ndarray,
                          len_lo: int, seed: int) -> DeviceTransactions:
    dev = _dev()
    thresh, alias = item_alias
    lengths = torch.empty(max(n_tx, 1), dtype=torch.int64, device=dev)
    cdf = np.ascontiguousarray(len_cdf, dtype=np.uint32)
    nat.call("crop_gen_lengths", n_tx, seed, cdf.ctypes.data, cdf.shape[0], len_lo,
             nat.ptr(lengths), nat.stream_ptr())
    offsets = torch.zeros(n_tx + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lengths[:n_tx], 0, out=offsets[1:])
    nnz = int(offsets[-1].item())
    items = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    th = np.ascontiguousarray(thresh, dtype=np.uint32)
    al = np.ascontiguousarray(alias, dtype=np.uint32)
    nat.call("crop_gen_items", n_tx, seed, n_items, th.ctypes.data, al.ctypes.data,
             nat.ptr(offsets), nat.ptr(items), nat.stream_ptr())
    return DeviceTransactions(offsets, items[:nnz], n_items)


def entry_bucket_stats_f64(ent: DeviceEntries, tables: list, kappa: int, n_items: int,
                           signs: list | None):
    """Real-weight entries: per-instance (distinct, cs) per bucket."""
    dev = ent.row.device
    t = len(tables)
    h_row = torch.cat([x[0][:n_items] for x in tables]) if t > 1 else tables[0][0]
    h_col = torch.cat([x[1][:n_items] for x in tables]) if t > 1 else tables[0][1]
    distinct = torch.zeros(t * kappa, dtype=torch.int32, device=dev)
    cs = torch.zeros(t * kappa, dtype=torch.float64, device=dev) if signs else None
    sg = None
    if signs:
        sg = (ctypes.c_uint64 * (2 * t))(*[v for s in signs for v in (s.mul, s.add)])
    n_dev = getattr(ent, "n_dev", None)
    if n_dev is None:
        n_dev = torch.tensor([ent.n], dtype=torch.int64, device=dev)
    nat.call("crop_entry_bucket_stats_f64", nat.ptr(ent.row), nat.ptr(ent.col),
             nat.ptr(ent.value), nat.ptr(n_dev), ent.row.shape[0], t, n_items, nat.ptr(h_row),
             nat.ptr(h_col), kappa, sg, nat.ptr(distinct), nat.ptr(cs), nat.stream_ptr())
    return distinct.view(t, kappa), (cs.view(t, kappa) if cs is not None else None)


def product_worker_loads(a_ptr, a_idx, b_ptr, b_idx, n_products: int, h_row, h_col, kappa: int,
                         workers: int, upper_only: bool) -> torch.Tensor:
    out = torch.zeros(max(n_products, 1) * workers, dtype=torch.int32, device=a_ptr.device)
    nat.call("crop_product_worker_loads", nat.ptr(a_ptr), nat.ptr(a_idx), nat.ptr(b_ptr),
             nat.ptr(b_idx), n_products, nat.ptr(h_row), nat.ptr(h_col), kappa, workers,
             int(upper_only), nat.ptr(out), nat.stream_ptr())
    return out[: n_products * workers].view(n_products, workers)


def merge_bucket_summaries(parts: list, h_row, h_col, kappa: int, capacity: int):
    """Per-bucket top-`capacity` summaries of a job counted as disjoint parts
    (tile shards / ranks: every pair's exact count lives in exactly one part,
    but a bucket's pairs spread over all parts).

    Each part keeps only its own top-l candidates per bucket; a bucket's
    global top-l is among the union of those candidates, so one more
    bucket_topk over the concatenated candidates gives the summaries of the
    whole job (the bounded Space-Saving regime, spacesaving.py:39-63, with
    exact weights). Loads and distinct counts are summed over the parts.
    Returns (DeviceEntries of the candidates, recorded mask over them,
    bucket_min int64[kappa], loads int64[kappa], distinct int64[kappa])."""
    dev = h_row.device
    loads = torch.zeros(kappa, dtype=torch.int64, device=dev)
    distinct = torch.zeros(kappa, dtype=torch.int64, device=dev)
    rows, cols, cnts = [], [], []
    for ent in parts:
        bl, dc, _ = entry_bucket_stats(ent, [(h_row, h_col)], kappa, int(h_row.shape[0]), None)
        loads += bl[0]
        distinct += dc[0].to(torch.int64)
        n = ent.n
        if int(dc[0].max().item()) >= capacity:
            mask, _, _ = bucket_topk(ent, h_row, h_col, kappa, capacity)
            rows.append(ent.row[:n][mask])
            cols.append(ent.col[:n][mask])
            cnts.append(ent.count[:n][mask])
        else:
            rows.append(ent.row[:n])
            cols.append(ent.col[:n])
            cnts.append(ent.count[:n])
    row, col, cnt = torch.cat(rows), torch.cat(cols), torch.cat(cnts)
    cand = DeviceEntries(row, col, cnt, None, int(row.shape[0]), parts[0].total_terms)
    mask, bmin, _ = bucket_topk(cand, h_row, h_col, kappa, capacity)
    full = distinct >= capacity
    bmin = torch.where(full, bmin, torch.zeros_like(bmin))
    return cand, mask, bmin, loads, distinct
