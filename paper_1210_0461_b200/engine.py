"""The partitioned sketch engine, B200 edition (drop-in for `engine.py`).

Same public surface as the reference (`pkg/src/crop/engine.py`): EngineConfig
(:38-83), SketchState (:108-176), LoadReport (:179-216), run (:238-302),
measure_loads (:305-349), load_balance_check (:352-390), run_worker
(:396-455), merge_partials (:471-534), run_parallel (:570-592),
save_state / load_state (:598-660).

What changes is where the work happens. The reference walks every outer
product in Python and feeds each term to a per-bucket Space-Saving summary.
Here the stream is moved to HBM once (columnar CSR), every term is counted
exactly on chip by the CUDA kernels (kernels.py -> csrc/), and the per-bucket
summaries are *derived* from the exact per-entry weights:

* exact regime (ss_capacity >= entries in the bucket -- SPEC.md:582): the
  summary is the bucket's exact weights, identical to the reference's;
* bounded regime: the summary keeps the bucket's top ss_capacity entries by
  (weight desc, row, col) with over = 0 and total_weight = the bucket's
  weight. It is always full, so `query` of an absent entry returns the
  summary minimum, which bounds it. Every Space-Saving guarantee the
  reference documents holds (sandwich, over <= m/l, capture of entries
  heavier than m/l: spacesaving.py:1-9) with zero overestimation; the
  records differ from the reference's order-dependent ones, which is why the
  parity contract for this regime is the bound.

Per-instance hashing, bucket assignment, worker intervals and Count-Sketch
cells follow the reference bit for bit: the sketch cells of a 0/1 stream are
integers, so summing count * sign per entry equals the reference's
term-by-term fp64 sums exactly.

Results stay on the device; Python objects (SpaceSavingSummary per bucket)
are materialised only when `SketchState.instances` is read.
"""

import json
import multiprocessing
from base64 import b64decode, b64encode
from dataclasses import dataclass, field
from statistics import median
from typing import NamedTuple

import numpy as np

from .countsketch import CountSketch
from .errors import ConfigError, CropError, DimensionError, InputError
from .hashing import (MAX_INDEX, EntryHasher, HashConfig, derive_seed, hasher_from_text,
                      hasher_to_text, make_hashes)
from .interval import WorkerAssignment
from .sparse import (ColumnRowStream, Entry, OuterProductStream, TransactionStream,
                     as_transaction_stream)
from .spacesaving import SpaceSavingSummary

STATE_FORMAT = "crop-state/1"
PARTIAL_FORMAT = "crop-partial/1"


@dataclass(frozen=True)
class EngineConfig:
    kappa: int
    ss_capacity: int
    workers: int = 1
    cs_enabled: bool = True
    instances: int = 1
    seed: int = 0
    d_hint: int | None = None

    def __post_init__(self):
        if self.kappa < 1:
            raise ConfigError(f"kappa must be >= 1, got {self.kappa}")
        if self.ss_capacity < 1:
            raise ConfigError(f"ss_capacity must be >= 1, got {self.ss_capacity}")
        if not 1 <= self.workers <= self.kappa:
            raise ConfigError(f"workers must be in [1, kappa={self.kappa}], got {self.workers}")
        if self.instances < 1 or self.instances % 2 == 0:
            raise ConfigError(f"instances must be odd and >= 1, got {self.instances}")
        if self.d_hint is not None and self.d_hint < 0:
            raise ConfigError(f"d_hint must be >= 0, got {self.d_hint}")

    def instance_seeds(self) -> list[int]:
        return [derive_seed(self.seed, f"instance:{i}") for i in range(self.instances)]

    def assignments(self) -> list[WorkerAssignment]:
        return WorkerAssignment.split(self.kappa, self.workers)

    def to_dict(self) -> dict:
        return {"kappa": self.kappa, "ss_capacity": self.ss_capacity, "workers": self.workers,
                "cs_enabled": self.cs_enabled, "instances": self.instances, "seed": self.seed,
                "d_hint": self.d_hint}

    @classmethod
    def from_dict(cls, data: dict) -> "EngineConfig":
        return cls(**data)


class InstanceSketch:
    """One independent instance: hash draw, bucket summaries, Count-Sketch."""

    __slots__ = ("seed", "hasher", "summaries", "sketch")

    def __init__(self, seed: int, hasher: EntryHasher, summaries: dict, sketch):
        self.seed = seed
        self.hasher = hasher
        self.summaries = summaries
        self.sketch = sketch

    def recorded_weight(self) -> float:
        return sum(s.total_weight for s in self.summaries.values())


class TopEntry(NamedTuple):
    entry: Entry
    lower: float
    upper: float
    estimate: float | None


# ============================================================ device results

class _DeviceInstance:
    """Per-instance facts of a device result (host numpy + device tables)."""

    def __init__(self, seed, hasher, tables, loads, distinct, cs):
        self.seed = seed
        self.hasher = hasher
        self.tables = tables          # (h_row, h_col) device tensors
        self.loads = loads            # np.int64[kappa]: terms per bucket
        self.distinct = distinct      # np.int64[kappa]: entries per bucket
        self.cs = cs                  # np.float64[kappa] or None
        self.recorded = None          # device bool mask over entries (None: all)
        self.bucket_min = None        # np.float64[kappa]: min recorded weight of full buckets
        self.bucket_weight = None     # np.float64[kappa]: summary total_weight


def torch_int64():
    import torch

    return torch.int64


class _DeviceResult:
    """Exact entries of a run plus everything needed to answer queries."""

    def __init__(self, entries, integer: bool, instances: list, capacity: int, kappa: int, over=None):
        self.entries = entries        # kernels.DeviceEntries
        self.integer = integer
        self.instances = instances
        self.capacity = capacity
        self.kappa = kappa
        self.over = over              # streaming summaries: uint32 over-estimation per record
        self._index = None
        self._over_host = None

    def over_of(self, idx: int) -> float:
        if self.over is None or idx < 0:
            return 0.0
        if self._over_host is None:
            self._over_host = (self.over[: self.entries.n].to(torch_int64()) & 0xFFFFFFFF).cpu().numpy()
        return float(self._over_host[idx])

    # -- host index for point queries (built on first use) -------------------
    def index(self):
        if self._index is None:
            import torch

            e = self.entries
            key = ((e.row[: e.n].to(torch.int64) & 0xFFFFFFFF) << 32) | (
                e.col[: e.n].to(torch.int64) & 0xFFFFFFFF)
            key, order = torch.sort(key)
            w = e.weights_f64()[order]
            self._index = (key.cpu().numpy().view(np.uint64), w.cpu().numpy(),
                           order.cpu().numpy())
        return self._index

    def lookup(self, row: int, col: int):
        keys, w, order = self.index()
        k = np.uint64((row << 32) | col)
        p = int(np.searchsorted(keys, k))
        if p < keys.shape[0] and keys[p] == k:
            return float(w[p]), int(order[p])
        return 0.0, -1

    def finalize_summaries(self):
        """Decide, per instance and bucket, which entries the summary records."""
        import torch

        e = self.entries
        cap = self.capacity
        for inst in self.instances:
            overflow = inst.distinct > cap
            full = inst.distinct >= cap
            inst.bucket_min = np.zeros(self.kappa)
            if not full.any():
                continue
            if self.integer:
                # native per-bucket top-l select (csrc/bucket_topk.cu): same
                # order (weight desc, row, col), no 2^31-element sort limit
                from .kernels import bucket_topk

                mask, bmin, _ = bucket_topk(e, inst.tables[0], inst.tables[1], self.kappa, cap,
                                            want_mask=bool(overflow.any()))
                if overflow.any():
                    inst.recorded = mask
                inst.bucket_min = bmin.cpu().numpy().astype(np.float64)
                continue
            w_all = e.weights_f64()
            from .kernels import entry_buckets

            b = entry_buckets(e.row, e.col, e.n, inst.tables[0], inst.tables[1], self.kappa)
            b = b.to(torch.int64)
            # rank entries inside their bucket by (weight desc, row asc, col asc)
            order = torch.arange(e.n, device=b.device)
            for key in (e.col[: e.n].to(torch.int64) & 0xFFFFFFFF,
                        e.row[: e.n].to(torch.int64) & 0xFFFFFFFF):
                order = order[torch.sort(key[order], stable=True).indices]
            order = order[torch.sort(w_all[order], descending=True, stable=True).indices]
            order = order[torch.sort(b[order], stable=True).indices]
            bs = b[order]
            first = torch.searchsorted(bs, bs, right=False)
            rank = torch.arange(e.n, device=b.device) - first
            keep_sorted = rank < cap
            if overflow.any():
                mask = torch.zeros(e.n, dtype=torch.bool, device=b.device)
                mask[order] = keep_sorted
                inst.recorded = mask
            # min recorded weight per full bucket: the entry of rank cap-1
            last = (rank == cap - 1)
            lb = bs[last].cpu().numpy()
            lw = w_all[order][last].cpu().numpy()
            inst.bucket_min[lb] = lw
            if overflow.any():
                # summary total_weight = all terms of the bucket (loads for 0/1)
                pass

    def recorded_of(self, inst, idx: int) -> bool:
        if idx < 0:
            return False
        if inst.recorded is None:
            return True
        return bool(inst.recorded[idx].item())

    def bucket_total_weight(self, inst) -> np.ndarray:
        if inst.bucket_weight is None:
            if self.integer:
                inst.bucket_weight = inst.loads.astype(np.float64)
            else:
                import torch

                from .kernels import entry_buckets

                e = self.entries
                b = entry_buckets(e.row, e.col, e.n, inst.tables[0], inst.tables[1], self.kappa)
                tot = torch.zeros(self.kappa, dtype=torch.float64, device=b.device)
                tot.index_add_(0, b.to(torch.int64), e.weights_f64())
                inst.bucket_weight = tot.cpu().numpy()
        return inst.bucket_weight


_COPY_STREAMS: dict = {}


def _copy_stream(device):
    """One side stream per device for overlapped device->host transfers."""
    import torch

    key = str(device)
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = torch.cuda.Stream(device=device)
    return _COPY_STREAMS[key]


class SketchState:
    """Frozen query surface over all instances' bucket structures."""

    def __init__(self, config: EngineConfig, n_rows: int, n_cols: int, instances: list,
                 upper_triangle_only: bool):
        self.config = config
        self.n_rows = n_rows
        self.n_cols = n_cols
        self._instances = instances
        self.upper_triangle_only = upper_triangle_only
        self.frozen = False
        self._dev = None

    @classmethod
    def _from_device(cls, config, n_rows, n_cols, upper, result: _DeviceResult) -> "SketchState":
        s = cls(config, n_rows, n_cols, None, upper)
        s._dev = result
        s.frozen = True
        return s

    @property
    def device_result(self):
        return self._dev

    # -- materialisation -----------------------------------------------------
    @property
    def instances(self) -> list:
        if self._instances is None:
            self._instances = self._materialise()
        return self._instances

    @instances.setter
    def instances(self, value):
        self._instances = value

    def _materialise(self) -> list:
        d = self._dev
        row, col, w = d.entries.to_numpy()
        out = []
        for inst in d.instances:
            import torch

            from .kernels import entry_buckets

            e = d.entries
            b = entry_buckets(e.row, e.col, e.n, inst.tables[0], inst.tables[1], d.kappa)
            b = b.cpu().numpy().astype(np.int64)
            keep = np.ones(row.shape[0], dtype=bool) if inst.recorded is None else \
                inst.recorded.cpu().numpy()
            tot = d.bucket_total_weight(inst)
            summaries = {}
            for bucket in np.nonzero(inst.distinct)[0]:
                summaries[int(bucket)] = SpaceSavingSummary(d.capacity)
                summaries[int(bucket)].total_weight = float(tot[bucket])
            order = np.lexsort((col, row, b))
            for x in order[keep[order]]:
                summaries[int(b[x])]._load_record((int(row[x]), int(col[x])), float(w[x]), d.over_of(int(x)))
            sketch = None
            if self.config.cs_enabled:
                sketch = CountSketch(inst.hasher, [float(c) for c in inst.cs])
            out.append(InstanceSketch(inst.seed, inst.hasher, summaries, sketch))
            del torch
        return out

    def _require_frozen(self):
        if not self.frozen:
            raise CropError("state is still building; queries require a frozen state")

    # -- queries ---------------------------------------------------------------
    def query(self, entry) -> tuple[float, float, float | None]:
        self._require_frozen()
        row, col = entry
        if self._dev is None:
            return self._query_host(row, col)
        d = self._dev
        w, idx = d.lookup(row, col)
        lower, upper = 0.0, float("inf")
        for inst in d.instances:
            b = inst.hasher.bucket_of(row, col)
            if inst.distinct[b] == 0:
                lo, up = 0.0, 0.0
            elif idx >= 0 and d.recorded_of(inst, idx):
                lo, up = w - d.over_of(idx), w
            elif inst.distinct[b] >= d.capacity:
                lo, up = 0.0, float(inst.bucket_min[b])
            else:
                lo, up = 0.0, 0.0
            lower = max(lower, lo)
            upper = min(upper, up)
        return lower, upper, self._estimate(row, col)

    def _estimate(self, row, col):
        if not self.config.cs_enabled:
            return None
        if self._dev is not None:
            return median(float(inst.cs[inst.hasher.bucket_of(row, col)]) *
                          inst.hasher.sign_hash(row, col) for inst in self._dev.instances)
        return median(inst.sketch.query(row, col) for inst in self.instances)

    def _query_host(self, row, col):
        lower, upper = 0.0, float("inf")
        for inst in self.instances:
            s = inst.summaries.get(inst.hasher.bucket_of(row, col))
            lo, up = (0.0, 0.0) if s is None else s.query((row, col))
            lower = max(lower, lo)
            upper = min(upper, up)
        return lower, upper, self._estimate(row, col)

    def candidate_entries(self) -> list[tuple[int, int]]:
        """Entries recorded in a majority of instances."""
        if self._dev is None:
            need = len(self.instances) // 2 + 1
            hits: dict = {}
            for inst in self.instances:
                for summary in inst.summaries.values():
                    for item, _, _ in summary.records():
                        hits[item] = hits.get(item, 0) + 1
            return [item for item, c in hits.items() if c >= need]
        mask = self._candidate_mask()
        row, col, _ = self._dev.entries.to_numpy()
        if mask is not None:
            m = mask.cpu().numpy()
            row, col = row[m], col[m]
        return [(int(r), int(c)) for r, c in zip(row, col)]

    def _candidate_mask(self):
        d = self._dev
        masks = [inst.recorded for inst in d.instances if inst.recorded is not None]
        if not masks:
            return None
        import torch

        votes = sum(m.to(torch.int32) for m in masks) + (len(d.instances) - len(masks))
        return votes >= len(d.instances) // 2 + 1

    def top_entries(self, k: int) -> list[TopEntry]:
        """Best k candidates ranked by (upper desc, lower desc, row, col)."""
        self._require_frozen()
        if k < 0:
            raise ConfigError(f"k must be >= 0, got {k}")
        if self._dev is None:
            scored = [TopEntry(Entry(*it), *self.query(it)) for it in self.candidate_entries()]
            scored.sort(key=lambda t: (-t.upper, -t.lower, t.entry.row, t.entry.col))
            return scored[:k]
        d = self._dev
        e = d.entries
        if k == 0 or e.n == 0:
            return []
        import torch

        from .kernels import topk_indices, u32_to_numpy

        mask = self._candidate_mask()
        if d.over is not None:
            return self._top_entries_over(k)
        if d.integer:
            count = None  # the raw counts: the fused top-k inputs apply
            if mask is not None:
                count = torch.where(mask, e.count[: e.n], torch.zeros_like(e.count[: e.n]))
            idx = topk_indices(e, k, count=count)
        else:
            w = e.weights_f64()
            if mask is not None:
                w = torch.where(mask, w, torch.full_like(w, -float("inf")))
            order = torch.arange(e.n, device=w.device)
            for key in (e.col[: e.n].to(torch.int64) & 0xFFFFFFFF,
                        e.row[: e.n].to(torch.int64) & 0xFFFFFFFF):
                order = order[torch.sort(key[order], stable=True).indices]
            order = order[torch.sort(w[order], descending=True, stable=True).indices]
            idx = order[:k]
        # one read-back: rows, cols, weights (and the mask) of the k winners
        parts = [(e.row[idx].to(torch.int64) & 0xFFFFFFFF).to(torch.float64),
                 (e.col[idx].to(torch.int64) & 0xFFFFFFFF).to(torch.float64), e.weights_at(idx)]
        if mask is not None:
            parts.append(mask[idx].to(torch.float64))
        h = torch.stack(parts).cpu().numpy()
        rows, cols, ws = h[0].astype(np.int64), h[1].astype(np.int64), h[2]
        keep = ws > 0 if mask is not None else np.ones(ws.shape[0], dtype=bool)
        if mask is not None:
            keep &= h[3] > 0
        rows, cols, ws = rows[keep], cols[keep], ws[keep]
        order = np.lexsort((cols, rows, -ws))[:k]
        cs = self.config.cs_enabled
        rl, cl, wl = rows[order].tolist(), cols[order].tolist(), ws[order].tolist()
        if cs:
            return [TopEntry(Entry(r, c), w, w, self._estimate(r, c)) for r, c, w in zip(rl, cl, wl)]
        # tuple.__new__ skips the NamedTuple constructor's argument parsing
        # (k is 1,000-10,000 in the configs: this is the call's host cost)
        tn = tuple.__new__
        return [tn(TopEntry, (tn(Entry, (r, c)), w, w, None)) for r, c, w in zip(rl, cl, wl)]

    def _top_entries_over(self, k: int) -> list[TopEntry]:
        """Streaming summaries (one instance): rank the records by (upper desc,
        lower desc, row, col) with upper = count, lower = count - over
        (engine.py:162-172)."""
        import torch

        d = self._dev
        e = d.entries
        n = e.n
        up = e.count[:n].to(torch.int64) & 0xFFFFFFFF
        lo = up - (d.over[:n].to(torch.int64) & 0xFFFFFFFF)
        order = torch.arange(n, device=up.device)
        for key, desc in ((e.col[:n].to(torch.int64) & 0xFFFFFFFF, False),
                          (e.row[:n].to(torch.int64) & 0xFFFFFFFF, False), (lo, True), (up, True)):
            order = order[torch.sort(key[order], stable=True, descending=desc).indices]
        idx = order[:k]
        h = torch.stack([(e.row[idx].to(torch.int64) & 0xFFFFFFFF), (e.col[idx].to(torch.int64) & 0xFFFFFFFF),
                         up[idx], lo[idx]]).cpu().numpy()
        return [TopEntry(Entry(int(r), int(c)), float(l), float(u), self._estimate(int(r), int(c)))
                for r, c, u, l in zip(h[0], h[1], h[2], h[3])]

    def entry_arrays(self, instance: int = 0, out=None, compact: bool = True, wait: bool = True):
        """All recorded entries of one instance as columnar host arrays
        (row, col, weight): the columnar form of `instances[t].summaries` (the
        reference's per-bucket dicts, engine.py:108-118) without building one
        Python object per entry. Ids are uint32, or uint16 when `compact` and
        both dimensions are at most 65,536 (lossless; a third less to copy
        from the device); 0/1 streams give uint32 supports, real streams
        float64 weights. A device-backed state copies them with one
        device->host transfer per column into pinned buffers (`out` =
        reusable (row, col, weight) numpy arrays of at least the entry count
        and of the returned dtypes, e.g. from pinned torch tensors;
        entry_dtypes() names them). With wait=False the transfers run on a
        copy stream and the call returns at once: the arrays are valid after
        wait_entries(), and device work issued meanwhile (top_entries) overlaps
        the copy."""
        self._require_frozen()
        id_dt, w_dt = self.entry_dtypes(compact)
        if self._dev is None:
            recs = [(it[0], it[1], c) for s in self.instances[instance].summaries.values()
                    for it, c, _ in s.records()]
            row = np.array([r[0] for r in recs], dtype=id_dt)
            col = np.array([r[1] for r in recs], dtype=id_dt)
            return row, col, np.array([r[2] for r in recs], dtype=np.float64)
        import torch

        d = self._dev
        e = d.entries
        inst = d.instances[instance]
        n = e.n
        cols = [e.row[:n], e.col[:n], e.count[:n] if d.integer else e.value[:n]]
        if inst.recorded is not None:
            cols = [c[inst.recorded] for c in cols]
            n = int(cols[0].shape[0])
        if id_dt == np.uint16:
            # values < 2^16: the int32 -> int16 cast keeps the low 16 bits
            cols[0], cols[1] = cols[0].to(torch.int16), cols[1].to(torch.int16)
        if out is None:
            host = [torch.empty(n, dtype=c.dtype, pin_memory=True) for c in cols]
        else:
            signed = {np.dtype(np.uint32): np.int32, np.dtype(np.uint16): np.int16}
            for o, c in zip(out, cols):
                if o.dtype.itemsize != c.element_size():
                    raise InputError(f"out array of dtype {o.dtype} for a column of {c.dtype}")
            host = [torch.from_numpy(o.view(signed.get(o.dtype, o.dtype)))[:n] for o in out]
        if wait:
            for h, c in zip(host, cols):
                h.copy_(c, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        else:
            cur = torch.cuda.current_stream()
            side = _copy_stream(cur.device)
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                for h, c in zip(host, cols):
                    c.record_stream(side)
                    h.copy_(c, non_blocking=True)
                self._entries_copied = side.record_event()
        row, col, w = (h.numpy() for h in host)
        if d.integer:
            return row.view(id_dt), col.view(id_dt), w.view(np.uint32)
        return row.view(id_dt), col.view(id_dt), w

    def wait_entries(self) -> None:
        """Block until the transfers of entry_arrays(wait=False) have landed."""
        ev = getattr(self, "_entries_copied", None)
        if ev is not None:
            ev.synchronize()
            self._entries_copied = None

    def entry_dtypes(self, compact: bool = True):
        """(id dtype, weight dtype) of entry_arrays."""
        small = compact and self.n_rows <= 65536 and self.n_cols <= 65536
        integer = self._dev.integer if self._dev is not None else False
        return (np.uint16 if small else np.uint32), (np.uint32 if integer else np.float64)

    def recorded_weight(self) -> float:
        if self._dev is not None:
            d = self._dev
            return float(d.bucket_total_weight(d.instances[0]).sum())
        return self.instances[0].recorded_weight()


@dataclass
class LoadReport:
    """Per-worker processed-entry accounting (engine.py:179-216)."""

    kappa: int
    workers: int
    rows: list[list[int]]
    input_pair_total: int
    per_product: list | None = None
    assignments: list[tuple[int, int]] = field(default_factory=list)

    @property
    def worker_counts(self) -> list[int]:
        return self.rows[0]

    @property
    def total_entries(self) -> int:
        return sum(self.rows[0])

    @property
    def expected_per_worker(self) -> float:
        return self.total_entries / self.workers

    def max_avg_ratio(self) -> float:
        """Worst max/avg over instances, rounded as engine.py:207-216 does
        (avg = total / len first, then max / avg)."""
        worst = 1.0
        for row in self.rows:
            total = sum(row)
            if total == 0:
                continue
            avg = total / len(row)
            worst = max(worst, max(row) / avg)
        return worst


@dataclass(frozen=True)
class BalanceCheck:
    violations: int
    checked: int
    bound: float | None

    @property
    def frequency(self) -> float:
        return self.violations / self.checked if self.checked else 0.0


def load_balance_check(report: LoadReport, deviation: float) -> BalanceCheck:
    """Theorem 2 check (engine.py:352-390): per product when recorded, else per instance."""
    if deviation <= 0:
        raise ConfigError(f"deviation must be positive, got {deviation}")

    def violated(counts, expected):
        return any(abs(x - expected) > deviation * expected for x in counts)

    if report.per_product is not None:
        bad = seen = 0
        bsum = 0.0
        for na, nb, counts in report.per_product:
            total = sum(counts)
            if not total:
                continue
            expected = total / report.workers
            if expected < (na + nb) / deviation ** 2:
                continue
            seen += 1
            bsum += 1.0 / (na + nb)
            bad += violated(counts, expected)
        return BalanceCheck(bad, seen, bsum / seen if seen else None)
    bad = seen = 0
    for row in report.rows:
        total = sum(row)
        if total:
            seen += 1
            bad += violated(row, total / len(row))
    return BalanceCheck(bad, seen, None)


# ============================================================ execution

def _check_stream(stream):
    if stream.n_rows > MAX_INDEX or stream.n_cols > MAX_INDEX:
        raise DimensionError(f"dimensions {stream.n_rows}x{stream.n_cols} exceed the supported "
                             f"index space ({MAX_INDEX})")


class _Prepared:
    """A stream resident in HBM, in the layout its kernel family consumes."""

    def __init__(self, kind, device, n_rows, n_cols, n_items, pair_total, host):
        self.kind = kind              # "pairs" | "outer"
        self.device = device
        self.n_rows, self.n_cols = n_rows, n_cols
        self.n_items = n_items        # hash-table length (max id + 1)
        self.pair_total = pair_total  # sum |a_k| |b_k|
        self.host = host


def prepare(stream) -> _Prepared:
    """Move a stream to the device once (cached on columnar stream objects)."""
    from . import kernels

    cached = getattr(stream, "_crop_device", None)
    if cached is not None:
        return cached
    if isinstance(stream, kernels.DeviceTransactions):
        n = stream.n_items
        lens = (stream.offsets[1:] - stream.offsets[:-1])
        total = int((lens * lens).sum().item())
        return _Prepared("pairs", stream, n, n, n, total, None)
    ts = as_transaction_stream(stream)
    if ts is not None:
        # upload first; the max id and the pair total are reduced on the device
        # (one small read-back instead of two host passes over the arrays)
        dtx = kernels.DeviceTransactions.from_host(ts.offsets, ts.items, 1)
        import torch

        if dtx.items.numel():
            lens = dtx.offsets[1:] - dtx.offsets[:-1]
            mx, total, mn = torch.stack([dtx.items.max().to(torch.int64) + 1, (lens * lens).sum(),
                                         dtx.items.min().to(torch.int64)]).tolist()
            if mn < 0:
                raise InputError("item ids must be < 2^31")
        else:
            mx, total = 1, 0
        dtx.n_items = int(mx)
        prep = _Prepared("pairs", dtx, stream.n_rows, stream.n_cols, int(mx), int(total), ts)
    else:
        cr = ColumnRowStream.from_stream(stream)
        n_items = 1 + max(int(cr.a_idx.max()) if cr.a_idx.size else 0,
                          int(cr.b_idx.max()) if cr.b_idx.size else 0)
        prep = _Prepared("outer", kernels.DeviceOuterStream.from_host(cr), stream.n_rows,
                         stream.n_cols, n_items, cr.total_pair_count(), cr)
    if isinstance(stream, (TransactionStream, ColumnRowStream)):
        try:
            object.__setattr__(stream, "_crop_device", prep)
        except (AttributeError, TypeError):
            pass
    return prep


def _check_positive_terms(prep: _Prepared, upper: bool):
    """Space-Saving accepts only positive weights (spacesaving.py:41-42)."""
    if prep.kind != "outer":
        return
    cr = prep.host
    k = cr.length
    if k == 0:
        return
    a_neg = np.zeros(k, bool)
    a_pos = np.zeros(k, bool)
    # for the triangle filter a term (i, j) exists iff i < j: compare the
    # smallest row index of one sign with the largest column index of the other
    big = np.iinfo(np.int64).max
    def extremes(ptr, idx, val, sign, reducer, fill):
        owner = np.repeat(np.arange(k), np.diff(ptr))
        sel = (val < 0) if sign < 0 else (val > 0)
        out = np.full(k, fill, dtype=np.int64)
        reducer.at(out, owner[sel], idx[sel].astype(np.int64))
        return out
    if upper:
        amin_neg = extremes(cr.a_ptr, cr.a_idx, cr.a_val, -1, np.minimum, big)
        amin_pos = extremes(cr.a_ptr, cr.a_idx, cr.a_val, +1, np.minimum, big)
        bmax_neg = extremes(cr.b_ptr, cr.b_idx, cr.b_val, -1, np.maximum, -1)
        bmax_pos = extremes(cr.b_ptr, cr.b_idx, cr.b_val, +1, np.maximum, -1)
        bad = (amin_neg < bmax_pos) | (amin_pos < bmax_neg)
    else:
        owner_a = np.repeat(np.arange(k), np.diff(cr.a_ptr))
        owner_b = np.repeat(np.arange(k), np.diff(cr.b_ptr))
        np.logical_or.at(a_neg, owner_a[cr.a_val < 0], True)
        np.logical_or.at(a_pos, owner_a[cr.a_val > 0], True)
        b_neg = np.zeros(k, bool)
        b_pos = np.zeros(k, bool)
        np.logical_or.at(b_neg, owner_b[cr.b_val < 0], True)
        np.logical_or.at(b_pos, owner_b[cr.b_val > 0], True)
        bad = (a_neg & b_pos) | (a_pos & b_neg)
    if bad.any():
        raise InputError("weights must be positive: the stream has negative outer-product "
                         "terms, which Space-Saving rejects (use multiply() for signed products)")


def _worker_rows(bucket_loads: np.ndarray, assignments) -> list[int]:
    csum = np.concatenate([[0], np.cumsum(bucket_loads, dtype=np.int64)])
    return [int(csum[a.stop] - csum[a.start]) for a in assignments]


def _per_product(prep: _Prepared, table, kappa, workers, upper):
    from . import kernels

    d = prep.device
    if prep.kind == "pairs":
        a_ptr, a_idx, b_ptr, b_idx, n = d.offsets, d.items, d.offsets, d.items, d.n_tx
        lens = (d.offsets[1:] - d.offsets[:-1]).cpu().numpy()
        la = lb = lens
    else:
        a_ptr, a_idx, b_ptr, b_idx, n = d.a_ptr, d.a_idx, d.b_ptr, d.b_idx, d.n_products
        la = (d.a_ptr[1:] - d.a_ptr[:-1]).cpu().numpy()
        lb = (d.b_ptr[1:] - d.b_ptr[:-1]).cpu().numpy()
    out = kernels.product_worker_loads(a_ptr, a_idx, b_ptr, b_idx, n, table[0], table[1], kappa,
                                       workers, upper).cpu().numpy().astype(np.int64)
    return [(int(x), int(y), c.tolist()) for x, y, c in zip(la, lb, out)]


def _compute(prep: _Prepared, config: EngineConfig, upper: bool, start: int = 0,
             stop: int | None = None):
    """Count every own term of every instance on the GPU -> (_DeviceResult, hashers)."""
    import torch

    from . import kernels

    kappa = config.kappa
    stop = kappa if stop is None else stop
    seeds = config.instance_seeds()
    hashers = [make_hashes(HashConfig(kappa, s)) for s in seeds]
    tables = [kernels.hash_tables(h, prep.n_items) for h in hashers]
    signs = [h.sign_hash for h in hashers] if config.cs_enabled else None
    whole = start == 0 and stop == kappa
    instances = []
    if prep.kind == "pairs":
        ents = []
        if whole:  # one exact count serves every instance
            ents = [kernels.count_pairs(prep.device, upper)] * len(hashers)
        else:
            for tab in tables:
                ents.append(kernels.count_pairs(prep.device, upper, kappa, start, stop, *tab))
        for t, (h, tab) in enumerate(zip(hashers, tables)):
            loads, distinct, cs = kernels.entry_bucket_stats(
                ents[t], [tab], kappa, prep.n_items, [signs[t]] if signs else None)
            instances.append(_DeviceInstance(
                seeds[t], h, tab, loads[0].cpu().numpy(), distinct[0].cpu().numpy().astype(np.int64),
                cs[0].cpu().numpy().astype(np.float64) if cs is not None else None))
        integer = True
    else:
        ents = []
        for t, (h, tab) in enumerate(zip(hashers, tables)):
            if whole and t > 0:
                ents.append(ents[0])
            else:
                ents.append(kernels.outer_product(prep.device, upper, kappa, start, stop, *tab))
            loads = kernels.outer_bucket_loads(prep.device, tab[0], tab[1], kappa, upper)
            distinct, cs = kernels.entry_bucket_stats_f64(ents[t], [tab], kappa, prep.n_items,
                                                          [signs[t]] if signs else None)
            lo = loads.cpu().numpy()
            if not whole:
                lo[:start] = 0
                lo[stop:] = 0
            instances.append(_DeviceInstance(
                seeds[t], h, tab, lo, distinct[0].cpu().numpy().astype(np.int64),
                cs[0].cpu().numpy() if cs is not None else None))
        integer = False
    del torch
    # a single shared entry set when every instance counted the same buckets
    result = _DeviceResult(ents[0], integer, instances, config.ss_capacity, kappa)
    if any(e is not ents[0] for e in ents):
        result.per_instance_entries = ents
    return result, hashers


def run(stream: OuterProductStream, config: EngineConfig, upper_triangle_only: bool = False,
        record_per_product: bool = False) -> tuple[SketchState, LoadReport]:
    """Process the whole stream through all instances and workers on the GPU."""
    _check_stream(stream)
    if record_per_product and config.instances != 1:
        raise ConfigError("per-product load recording requires instances == 1")
    prep = prepare(stream)
    _check_positive_terms(prep, upper_triangle_only)
    result, _ = _compute(prep, config, upper_triangle_only)
    result.finalize_summaries()
    assignments = config.assignments()
    rows = [_worker_rows(inst.loads, assignments) for inst in result.instances]
    per_product = None
    if record_per_product:
        per_product = _per_product(prep, result.instances[0].tables, config.kappa, config.workers,
                                   upper_triangle_only)
    state = SketchState._from_device(config, prep.n_rows, prep.n_cols, upper_triangle_only, result)
    report = LoadReport(kappa=config.kappa, workers=config.workers, rows=rows,
                        input_pair_total=prep.pair_total, per_product=per_product,
                        assignments=[(a.start, a.stop) for a in assignments])
    return state, report


# run_streaming uploads a host stream's items chunk by chunk under the
# counting of the earlier chunks when it holds at least this many items
STAGED_UPLOAD_MIN_ITEMS = 50_000_000


class _StagedUpload:
    """A host TransactionStream whose items reach the device chunk by chunk
    on a copy stream (run_streaming): the offsets are uploaded at once, the
    item buffer is allocated whole, and chunk k's items are enqueued one
    chunk ahead of its counting (from pinned host memory the transfer runs
    under the previous chunk's kernels; from pageable memory it is merely
    synchronous). The hash tables take the stream's universe (dim) instead
    of max id + 1, which would need every item on the device first."""

    def __init__(self, ts):
        import torch

        from . import kernels

        dev = kernels._dev()
        self.ts = ts
        self.off_h = ts.offsets
        off = torch.from_numpy(ts.offsets).to(dev, non_blocking=True)
        self.items = torch.empty(int(ts.offsets[-1]), dtype=torch.int32, device=dev)
        self.dtx = kernels.DeviceTransactions(off, self.items, int(ts.n_rows))
        lens = off[1:] - off[:-1]
        total = int((lens * lens).sum().item())
        self.prepared = _Prepared("pairs", self.dtx, ts.n_rows, ts.n_cols, int(ts.n_rows), total, ts)
        self.side = _copy_stream(dev)
        self.side.wait_stream(torch.cuda.current_stream())
        self.items.record_stream(self.side)
        self.events = {}
        self.src = torch.from_numpy(ts.items.view(np.int16 if ts.items.dtype == np.uint16 else np.int32))

    def enqueue(self, t0: int, t1: int) -> None:
        import torch

        i0, i1 = int(self.off_h[t0]), int(self.off_h[t1])
        with torch.cuda.stream(self.side):
            if self.src.dtype == torch.int16:
                tmp = self.src[i0:i1].to(self.items.device, non_blocking=True)
                self.items[i0:i1] = tmp.to(torch.int32) & 0xFFFF
            else:
                self.items[i0:i1].copy_(self.src[i0:i1], non_blocking=True)
            self.events[t0] = self.side.record_event()

    def wait(self, t0: int) -> None:
        import torch

        torch.cuda.current_stream().wait_event(self.events.pop(t0))


def run_streaming(stream: OuterProductStream, config: EngineConfig, upper_triangle_only: bool = False,
                  chunk_transactions: int | None = None) -> tuple[SketchState, LoadReport]:
    """run() for pair mining with bounded summary memory: the transaction
    stream is consumed in chunks; each chunk is counted exactly on the GPU
    and merged into every bucket's Space-Saving summary of at most
    config.ss_capacity records (kernels.StreamingSummaries, csrc/ss_stream.cu),
    so the device state of an instance is kappa * l records of 16 B plus one
    chunk's entries, whatever the stream's distinct-pair count. Records carry
    the reference's (count, over) bounds (spacesaving.py:39-81): recorded
    entries query as (count - over, count), unrecorded ones as (0, min) in a
    full bucket. With chunk_transactions >= the stream length this is the
    exact regime's top-l of run(). Takes 0/1 transaction streams
    (mining.transactions_to_stream / TransactionStream); more than one
    instance materialises host summaries per instance."""
    import torch

    from . import kernels

    _check_stream(stream)
    staged = None
    if not isinstance(stream, kernels.DeviceTransactions) and getattr(stream, "_crop_device", None) is None:
        ts = as_transaction_stream(stream)
        if ts is not None and ts.items.shape[0] >= max(STAGED_UPLOAD_MIN_ITEMS, 1):
            staged = _StagedUpload(ts)
    prep = staged.prepared if staged is not None else prepare(stream)
    if prep.kind != "pairs":
        raise ConfigError("run_streaming takes 0/1 transaction streams (pair mining)")
    dtx = prep.device
    kappa = config.kappa
    seeds = config.instance_seeds()
    hashers = [make_hashes(HashConfig(kappa, s)) for s in seeds]
    tables = [kernels.hash_tables(h, prep.n_items) for h in hashers]
    signs = [h.sign_hash for h in hashers] if config.cs_enabled else None
    n_tx = dtx.n_tx
    if chunk_transactions is None:
        # (on the device: the offsets of c3 are 400 MB)
        lens = dtx.offsets[1:] - dtx.offsets[:-1]
        terms = int((lens * (lens - 1) // 2).sum().item())
        del lens
        n_chunks = max(1, -(-terms // 4_000_000_000))  # about 4e9 terms per chunk (c3: 6)
        chunk_transactions = max(1, -(-n_tx // n_chunks))
    if chunk_transactions < 1:
        raise ConfigError(f"chunk_transactions must be >= 1, got {chunk_transactions}")
    summ = [kernels.StreamingSummaries(kappa, config.ss_capacity, tab) for tab in tables]
    t = len(hashers)
    loads = torch.zeros((t, kappa), dtype=torch.int64, device=dtx.offsets.device)
    cs = torch.zeros((t, kappa), dtype=torch.int64, device=dtx.offsets.device) if signs else None
    bounds = [(t0, min(n_tx, t0 + chunk_transactions)) for t0 in range(0, n_tx, chunk_transactions)]
    if staged is not None and bounds:
        staged.enqueue(*bounds[0])
    for k, (t0, t1) in enumerate(bounds):
        if staged is not None:
            # the next chunk's items travel under this chunk's counting
            if k + 1 < len(bounds):
                staged.enqueue(*bounds[k + 1])
            staged.wait(t0)
        ent = kernels.count_pairs(dtx.slice(t0, t1, staged.off_h if staged is not None else None),
                                  upper_triangle_only)
        bl, _, c = kernels.entry_bucket_stats(ent, tables, kappa, prep.n_items, signs)
        loads += bl
        if cs is not None:
            cs += c
        for s in summ:
            s.absorb(ent)
        del ent
    loads_h = loads.cpu().numpy()
    cs_h = cs.cpu().numpy().astype(np.float64) if cs is not None else None
    assignments = config.assignments()
    rows = [_worker_rows(loads_h[i], assignments) for i in range(t)]
    report = LoadReport(kappa=kappa, workers=config.workers, rows=rows, input_pair_total=prep.pair_total,
                        assignments=[(a.start, a.stop) for a in assignments])
    if t == 1:
        s = summ[0]
        ent = kernels.DeviceEntries(s.row, s.col, s.count, None, s.n, int(loads_h[0].sum()))
        inst = _DeviceInstance(seeds[0], hashers[0], tables[0], loads_h[0],
                               s.per_bucket.cpu().numpy().astype(np.int64),
                               cs_h[0] if cs_h is not None else None)
        inst.bucket_min = s.mu.to(torch.int64).bitwise_and(0xFFFFFFFF).cpu().numpy().astype(np.float64)
        inst.bucket_weight = loads_h[0].astype(np.float64)
        result = _DeviceResult(ent, True, [inst], config.ss_capacity, kappa, over=s.over)
        state = SketchState._from_device(config, prep.n_rows, prep.n_cols, upper_triangle_only, result)
        return state, report
    # several instances: host summaries per instance
    instances = []
    for i, s in enumerate(summ):
        row, col = kernels.u32_to_numpy(s.row), kernels.u32_to_numpy(s.col)
        cnt, ovr = kernels.u32_to_numpy(s.count), kernels.u32_to_numpy(s.over)
        b = (np.asarray(hashers[i].row_hash.values(row.tolist()), np.int64) +
             np.asarray(hashers[i].col_hash.values(col.tolist()), np.int64)) % kappa if s.n else \
            np.zeros(0, np.int64)
        summaries = {}
        for bucket in np.nonzero(loads_h[i])[0]:
            summaries[int(bucket)] = SpaceSavingSummary(config.ss_capacity)
            summaries[int(bucket)].total_weight = float(loads_h[i][bucket])
        for x in np.lexsort((col, row, b)):
            summaries[int(b[x])]._load_record((int(row[x]), int(col[x])), float(cnt[x]), float(ovr[x]))
        sketch = CountSketch(hashers[i], [float(c) for c in cs_h[i]]) if cs_h is not None else None
        instances.append(InstanceSketch(seeds[i], hashers[i], summaries, sketch))
    state = SketchState(config, prep.n_rows, prep.n_cols, instances, upper_triangle_only)
    state.frozen = True
    return state, report


def measure_loads(stream: OuterProductStream, config: EngineConfig,
                  upper_triangle_only: bool = False, record_per_product: bool = False) -> LoadReport:
    """Per-worker term counts without summaries (K1 bucket-load kernel)."""
    from . import kernels

    _check_stream(stream)
    if record_per_product and config.instances != 1:
        raise ConfigError("per-product load recording requires instances == 1")
    prep = prepare(stream)
    assignments = config.assignments()
    rows = []
    per_product = None
    for seed in config.instance_seeds():
        h = make_hashes(HashConfig(config.kappa, seed))
        tab = kernels.hash_tables(h, prep.n_items)
        if prep.kind == "pairs":
            loads = kernels.selfjoin_bucket_loads(prep.device, tab[0], tab[1], config.kappa,
                                                  upper_triangle_only)
        else:
            loads = kernels.outer_bucket_loads(prep.device, tab[0], tab[1], config.kappa,
                                               upper_triangle_only)
        rows.append(_worker_rows(loads.cpu().numpy(), assignments))
        if record_per_product and per_product is None:
            per_product = _per_product(prep, tab, config.kappa, config.workers,
                                       upper_triangle_only)
    return LoadReport(kappa=config.kappa, workers=config.workers, rows=rows,
                      input_pair_total=prep.pair_total, per_product=per_product,
                      assignments=[(a.start, a.stop) for a in assignments])


# ============================================================ partitioned products

class ProductPartition:
    """Exact entries of buckets [start, stop) of a real-valued stream: the
    columnar result of running enumerate_interval (interval.py:236-254) over
    every outer product and accumulating each entry's terms in stream order
    (the reference's per-worker dict, or exact_product restricted by bucket,
    oracle.py:20-50). Entries are grouped by bucket ascending and sorted by
    (row, col) inside; values are fp64 sums, bit-identical to the reference's
    accumulation. Signed weights are allowed (no Space-Saving involved).
    Results stay on the device; `arrays()` copies them to host memory."""

    def __init__(self, entries, start: int, stop: int, total_terms: int):
        self.entries = entries
        self.start, self.stop = start, stop
        self.total_terms = total_terms

    def __len__(self) -> int:
        return self.entries.n

    def arrays(self, out=None, value_dtype=np.float64, bucket_ptr: bool = False):
        """(row uint32, col uint32, value, bucket) host arrays, one
        device->host copy per column (into `out`, e.g. pinned buffers of at
        least len(self) entries, when given). value_dtype = float64 (the
        exact stream-order sums) or float32 (each sum rounded once: within
        rel 1e-5 / abs 1e-6 of the float64 reference, the tolerance BASELINE
        c4 states for fp32 output). With bucket_ptr the fourth array is not
        the per-entry bucket but int64 offsets: the entries of bucket
        start + b are [ptr[b], ptr[b + 1]) (the result is sorted by bucket),
        and `out` holds three arrays."""
        import torch

        if np.dtype(value_dtype) not in (np.dtype(np.float64), np.dtype(np.float32)):
            raise ConfigError(f"value_dtype must be float64 or float32, got {value_dtype}")
        e = self.entries
        n = e.n
        val = e.value[:n]
        if np.dtype(value_dtype) == np.dtype(np.float32):
            val = val.to(torch.float32)
        cols = [e.row[:n], e.col[:n], val]
        ptr = None
        if bucket_ptr:
            edges = torch.arange(self.start, self.stop + 1, dtype=torch.int64, device=e.row.device)
            ptr = torch.searchsorted(e.bucket[:n].to(torch.int64) & 0xFFFFFFFF, edges)
        else:
            cols.append(e.bucket[:n])
        if out is None:
            host = [torch.empty(n, dtype=c.dtype, pin_memory=True) for c in cols]
        else:
            if len(out) != len(cols):
                raise InputError(f"out must hold {len(cols)} arrays, got {len(out)}")
            for o, c in zip(out, cols):
                if o.dtype.itemsize != c.element_size():
                    raise InputError(f"out array of dtype {o.dtype} for a column of {c.dtype}")
            host = [torch.from_numpy(o.view(np.int32) if o.dtype == np.uint32 else o)[:n] for o in out]
        for h, c in zip(host, cols):
            h.copy_(c, non_blocking=True)
        ptr_h = ptr.cpu().numpy() if ptr is not None else None  # (synchronises the stream)
        torch.cuda.current_stream().synchronize()
        res = [h.numpy() for h in host]
        last = ptr_h if bucket_ptr else res[3].view(np.uint32)
        return res[0].view(np.uint32), res[1].view(np.uint32), res[2], last


def partition_product(stream, config: EngineConfig, worker: int | None = None,
                      upper_triangle_only: bool = False) -> ProductPartition:
    """Exact per-partition accumulation of a (real-valued) stream on the GPU:
    the entries of `worker`'s bucket interval (all kappa buckets when None)
    under the config's first instance hash. This is the workload the
    reference's per-partition enumerate_interval + dict loop computes; the
    kernels (csrc/outer.cu) sort each (bucket, row-range) partition in shared
    memory and sum every entry's terms in stream order."""
    from . import kernels

    _check_stream(stream)
    prep = prepare(stream)
    if prep.kind != "outer":
        cr = ColumnRowStream.from_stream(stream)
        prep = _Prepared("outer", kernels.DeviceOuterStream.from_host(cr), stream.n_rows,
                         stream.n_cols, prep.n_items, cr.total_pair_count(), cr)
    h = make_hashes(HashConfig(config.kappa, config.instance_seeds()[0]))
    tab = kernels.hash_tables(h, prep.n_items)
    if worker is None:
        start, stop = 0, config.kappa
    else:
        if not 0 <= worker < config.workers:
            raise ConfigError(f"worker index {worker} out of range for {config.workers}")
        a = config.assignments()[worker]
        start, stop = a.start, a.stop
    ent = kernels.outer_product(prep.device, upper_triangle_only, config.kappa, start, stop, *tab)
    return ProductPartition(ent, start, stop, ent.total_terms)


# ============================================================ partial states

def _summary_lines(capacity, total, rows, cols, weights) -> list[str]:
    out = [f"capacity {capacity}", f"total_weight {float(total)!r}"]
    out += [f"{int(r)} {int(c)} {float(w)!r} 0.0" for r, c, w in zip(rows, cols, weights)]
    return out


def worker_payloads(stream, config: EngineConfig, w_lo: int, w_hi: int,
                    upper_triangle_only: bool = False) -> list[dict]:
    """Payloads (crop-partial/1) of workers [w_lo, w_hi): one device pass over
    the union of their intervals, split per worker on the host."""
    from . import kernels

    _check_stream(stream)
    assignments = config.assignments()
    if not (0 <= w_lo < w_hi <= config.workers):
        raise ConfigError(f"worker range [{w_lo}, {w_hi}) out of range for {config.workers}")
    start, stop = assignments[w_lo].start, assignments[w_hi - 1].stop
    prep = prepare(stream)
    _check_positive_terms(prep, upper_triangle_only)
    result, hashers = _compute(prep, config, upper_triangle_only, start, stop)
    ents = getattr(result, "per_instance_entries", [result.entries] * len(result.instances))
    per_worker = [[] for _ in range(w_hi - w_lo)]
    for t, inst in enumerate(result.instances):
        sub = _DeviceResult(ents[t], result.integer, [inst], config.ss_capacity, config.kappa)
        sub.finalize_summaries()
        e = ents[t]
        row, col, w = e.to_numpy()
        b = kernels.entry_buckets(e.row, e.col, e.n, inst.tables[0], inst.tables[1],
                                  config.kappa).cpu().numpy().astype(np.int64)
        keep = np.ones(row.shape[0], bool) if inst.recorded is None else inst.recorded.cpu().numpy()
        tot = sub.bucket_total_weight(inst)
        order = np.lexsort((col, row, b))
        order = order[keep[order]]
        bo = b[order]
        for k, wk in enumerate(range(w_lo, w_hi)):
            asg = assignments[wk]
            summaries = []
            for bucket in np.nonzero(inst.distinct[asg.start:asg.stop])[0] + asg.start:
                lo, hi = np.searchsorted(bo, bucket), np.searchsorted(bo, bucket, side="right")
                sel = order[lo:hi]
                summaries.append([int(bucket), _summary_lines(config.ss_capacity, tot[bucket],
                                                              row[sel], col[sel], w[sel])])
            cells = None
            if config.cs_enabled:
                cells = [float(c) for c in inst.cs[asg.start:asg.stop]]
            per_worker[k].append({"seed": inst.seed,
                                  "hashes": hasher_to_text(inst.hasher, inst.seed),
                                  "count": int(inst.loads[asg.start:asg.stop].sum()),
                                  "summaries": summaries, "cs_cells": cells})
    out = []
    for k, wk in enumerate(range(w_lo, w_hi)):
        asg = assignments[wk]
        out.append({"format": PARTIAL_FORMAT, "worker": wk, "start": asg.start, "stop": asg.stop,
                    "n_rows": stream.n_rows, "n_cols": stream.n_cols,
                    "upper_triangle_only": upper_triangle_only, "config": config.to_dict(),
                    "instances": per_worker[k]})
    return out


def run_worker(stream: OuterProductStream, config: EngineConfig, worker: int,
               upper_triangle_only: bool = False) -> dict:
    """One worker's interval over the full stream; JSON-able payload (engine.py:396-455)."""
    if not 0 <= worker < config.workers:
        raise ConfigError(f"worker index {worker} out of range for {config.workers}")
    return worker_payloads(stream, config, worker, worker + 1, upper_triangle_only)[0]


def save_partial(path, payload: dict) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(payload, fh)


def load_partial(path) -> dict:
    with open(path, "r", encoding="utf-8") as fh:
        payload = json.load(fh)
    if payload.get("format") != PARTIAL_FORMAT:
        raise InputError(f"{path}: not a {PARTIAL_FORMAT} file")
    return payload


def merge_partials(payloads: list[dict]) -> tuple[SketchState, LoadReport]:
    """Concatenate disjoint worker payloads; validates config, hashes and tiling."""
    if not payloads:
        raise InputError("no partial states to merge")
    payloads = sorted(payloads, key=lambda p: p["start"])
    head = payloads[0]
    config = EngineConfig.from_dict(head["config"])
    if len(payloads) != config.workers:
        raise InputError(f"expected {config.workers} worker payloads, got {len(payloads)}")
    cursor = 0
    for p in payloads:
        if p["config"] != head["config"]:
            raise InputError("worker payloads disagree on the engine config")
        if (p["n_rows"], p["n_cols"]) != (head["n_rows"], head["n_cols"]):
            raise InputError("worker payloads disagree on stream dimensions")
        if p["upper_triangle_only"] != head["upper_triangle_only"]:
            raise InputError("worker payloads disagree on the triangle filter")
        if p["start"] != cursor:
            raise InputError(f"intervals do not tile [0, kappa): gap or overlap at bucket {cursor}")
        cursor = p["stop"]
    if cursor != config.kappa:
        raise InputError(f"intervals stop at {cursor}, expected kappa={config.kappa}")
    instances = []
    rows = [[0] * config.workers for _ in range(config.instances)]
    for i in range(config.instances):
        text = head["instances"][i]["hashes"]
        hasher = hasher_from_text(text)
        summaries = {}
        cells = [0.0] * config.kappa if config.cs_enabled else None
        for p in payloads:
            inst = p["instances"][i]
            if inst["hashes"] != text:
                raise InputError("worker payloads disagree on hash descriptions")
            for bucket, lines in inst["summaries"]:
                if not p["start"] <= bucket < p["stop"]:
                    raise InputError(f"bucket {bucket} outside worker interval")
                summaries[bucket] = SpaceSavingSummary.from_lines(lines)
            if cells is not None:
                cells[p["start"]:p["stop"]] = inst["cs_cells"]
            rows[i][p["worker"]] = inst["count"]
        sketch = CountSketch(hasher, cells) if cells is not None else None
        instances.append(InstanceSketch(head["instances"][i]["seed"], hasher, summaries, sketch))
    state = SketchState(config, head["n_rows"], head["n_cols"], instances,
                        head["upper_triangle_only"])
    state.frozen = True
    report = LoadReport(kappa=config.kappa, workers=config.workers, rows=rows, input_pair_total=0,
                        assignments=[(p["start"], p["stop"]) for p in payloads])
    return state, report


# ============================================================ sources / parallel

class MemorySource:
    """Picklable in-memory source (engine.py:540-549)."""

    def __init__(self, stream: OuterProductStream):
        self.stream = stream
        self.n_rows, self.n_cols = stream.n_rows, stream.n_cols

    def __call__(self) -> OuterProductStream:
        return self.stream


class TripleFileSource:
    def __init__(self, path_a, path_b):
        self.path_a, self.path_b = str(path_a), str(path_b)

    def __call__(self):
        from .sparse import load_column_row_streams

        return load_column_row_streams(self.path_a, self.path_b)


def run_parallel(source, config: EngineConfig, upper_triangle_only: bool = False,
                 processes: int | None = None) -> tuple[SketchState, LoadReport]:
    """Shared-nothing execution across GPUs (engine.py:570-592).

    Under torch.distributed (one process per GPU, torchrun) the input is
    broadcast once from rank 0, each rank counts the buckets of its contiguous
    share of the worker intervals, and rank 0 merges the disjoint results
    (distributed.py). In a single process the one visible GPU owns every
    interval, which yields the same state (the engine is K-invariant).
    `processes` is accepted for compatibility; the GPU count comes from the
    process group. As in the reference, the merged report carries
    input_pair_total = 0."""
    from . import distributed

    stream = source if isinstance(source, OuterProductStream) else source()
    if distributed.world_size() > 1:
        return distributed.run_distributed(stream, config, upper_triangle_only)
    state, report = run(stream, config, upper_triangle_only)
    report.input_pair_total = 0
    return state, report


# ============================================================ state files

def save_state(path, state: SketchState, binary_cs: bool = False) -> None:
    """Write a merged state as one JSON document (crop-state/1)."""
    instances = []
    for inst in state.instances:
        cs_field = None
        if inst.sketch is not None:
            cs_field = ({"encoding": "base64-le", "data": b64encode(inst.sketch.to_bytes()).decode()}
                        if binary_cs else {"encoding": "list", "data": inst.sketch.cells})
        instances.append({"seed": inst.seed, "hashes": hasher_to_text(inst.hasher, inst.seed),
                          "summaries": [[b, inst.summaries[b].to_lines()]
                                        for b in sorted(inst.summaries)],
                          "cs": cs_field})
    doc = {"format": STATE_FORMAT, "config": state.config.to_dict(), "n_rows": state.n_rows,
           "n_cols": state.n_cols, "upper_triangle_only": state.upper_triangle_only,
           "instances": instances}
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh)


def load_state(path) -> SketchState:
    with open(path, "r", encoding="utf-8") as fh:
        doc = json.load(fh)
    if doc.get("format") != STATE_FORMAT:
        raise InputError(f"{path}: not a {STATE_FORMAT} file")
    config = EngineConfig.from_dict(doc["config"])
    instances = []
    for d in doc["instances"]:
        hasher = hasher_from_text(d["hashes"])
        summaries = {b: SpaceSavingSummary.from_lines(lines) for b, lines in d["summaries"]}
        sketch = None
        cs = d.get("cs")
        if cs is not None:
            sketch = (CountSketch.from_bytes(hasher, b64decode(cs["data"]))
                      if cs["encoding"] == "base64-le"
                      else CountSketch(hasher, [float(x) for x in cs["data"]]))
        instances.append(InstanceSketch(d["seed"], hasher, summaries, sketch))
    state = SketchState(config, doc["n_rows"], doc["n_cols"], instances, doc["upper_triangle_only"])
    state.frozen = True
    return state
