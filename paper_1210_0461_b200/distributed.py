"""Multi-GPU execution: broadcast the input once, count disjoint intervals, gather.

The paper's processors each hold the whole input and never communicate
after the broadcast; the reference emulates this
with one OS process per worker and a pickled/JSON merge (engine.py:540-592).
Here one process per GPU (torchrun) is the worker pool:

1. rank 0 broadcasts the columnar stream (CSR offsets/items, or CSC/CSR with
   values) with `torch.distributed.broadcast` -- NCCL over NVLink on B200,
   gloo on CPU in the tests;
2. rank r owns the contiguous block of worker intervals
   [r*W/G, (r+1)*W/G) and counts only the buckets of that block on its GPU
   (no communication while counting);
3. the disjoint per-worker payloads are gathered to rank 0 and merged with
   `merge_partials`, which validates the tiling of [0, kappa).

Because bucket ownership depends only on (i, j) and the seed, the merged
state is identical for every G (the reference's K-invariance).
The per-rank compute function is injectable so the CPU tests can drive the
same orchestration with the oracle (tests/test_distributed.py).
"""

import numpy as np


def _dist():
    import torch.distributed as dist

    return dist


def world_size() -> int:
    dist = _dist()
    return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1


def rank() -> int:
    dist = _dist()
    return dist.get_rank() if dist.is_available() and dist.is_initialized() else 0


def rank_workers(workers: int, r: int, world: int) -> tuple[int, int]:
    """Contiguous worker block [lo, hi) of rank r (empty when world > workers)."""
    return r * workers // world, (r + 1) * workers // world


def _device_for_backend():
    import torch

    dist = _dist()
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_arrays(arrays: dict | None, src: int = 0) -> dict:
    """Broadcast named 1-D numpy arrays from `src` (shapes first, then data)."""
    import torch

    dist = _dist()
    dev = _device_for_backend()
    me = dist.get_rank()
    names = sorted(arrays) if me == src else None
    obj = [names, {k: (str(arrays[k].dtype), arrays[k].shape[0]) for k in names}
           if me == src else None]
    dist.broadcast_object_list(obj, src=src)
    names, meta = obj
    out = {}
    for k in names:
        dtype, n = meta[k]
        np_dt = np.dtype(dtype)
        view = {np.dtype(np.uint32): np.int32, np.dtype(np.uint64): np.int64}.get(np_dt, np_dt)
        if me == src:
            t = torch.from_numpy(np.ascontiguousarray(arrays[k]).view(view)).to(dev)
        else:
            t = torch.empty(n, dtype=getattr(torch, np.dtype(view).name), device=dev)
        dist.broadcast(t, src=src)
        out[k] = t.cpu().numpy().view(np_dt)
    return out


def _stream_arrays(stream) -> dict:
    from .sparse import ColumnRowStream, as_transaction_stream

    ts = as_transaction_stream(stream)
    if ts is not None:
        return {"kind": np.array([0]), "dim": np.array([stream.n_rows], dtype=np.int64),
                "offsets": ts.offsets, "items": ts.items}
    cr = ColumnRowStream.from_stream(stream)
    return {"kind": np.array([1]), "dim": np.array([cr.n_rows, cr.n_cols], dtype=np.int64),
            "a_ptr": cr.a_ptr, "a_idx": cr.a_idx, "a_val": cr.a_val,
            "b_ptr": cr.b_ptr, "b_idx": cr.b_idx, "b_val": cr.b_val}


def _stream_from_arrays(arr: dict):
    from .sparse import ColumnRowStream, TransactionStream

    if int(arr["kind"][0]) == 0:
        return TransactionStream(int(arr["dim"][0]), arr["offsets"], arr["items"], validate=False)
    return ColumnRowStream(int(arr["dim"][0]), int(arr["dim"][1]), arr["a_ptr"], arr["a_idx"],
                           arr["a_val"], arr["b_ptr"], arr["b_idx"], arr["b_val"])


def run_distributed(stream, config, upper_triangle_only: bool = False, compute=None, src: int = 0):
    """SPMD body of run_parallel. Returns (state, report) on rank `src`,
    (None, None) elsewhere. Without `compute` and with one instance the whole
    path stays on the GPUs (run_distributed_device); otherwise
    `compute(stream, config, w_lo, w_hi, upper)` returns the crop-partial/1
    payloads of a worker block (default: the GPU engine's worker_payloads),
    gathered to `src` and merged with merge_partials."""
    from .engine import merge_partials, worker_payloads

    dist = _dist()
    if compute is None and config.instances == 1 and config.workers >= dist.get_world_size():
        return run_distributed_device(stream, config, upper_triangle_only, src)
    dist = _dist()
    me, world = dist.get_rank(), dist.get_world_size()
    local = _stream_from_arrays(broadcast_arrays(_stream_arrays(stream) if me == src else None,
                                                 src=src))
    compute = compute or worker_payloads
    lo, hi = rank_workers(config.workers, me, world)
    payloads = compute(local, config, lo, hi, upper_triangle_only) if hi > lo else []
    gathered = [None] * world if me == src else None
    dist.gather_object(payloads, gathered, dst=src)
    if me != src:
        return None, None
    return merge_partials([p for part in gathered for p in part])


def _send(t, dst: int):
    """Point-to-point send on the group's device (host copy under gloo)."""
    dist = _dist()
    dist.send(t if dist.get_backend() == "nccl" or t.device.type == "cpu" else t.cpu(), dst)


def _recv(t, src: int):
    dist = _dist()
    if dist.get_backend() == "nccl" or t.device.type == "cpu":
        dist.recv(t, src)
        return
    h = torch_empty_like_cpu(t)
    dist.recv(h, src)
    t.copy_(h)


def torch_empty_like_cpu(t):
    import torch

    return torch.empty(t.shape, dtype=t.dtype, device="cpu")


def _gather_cat(t, sizes: list, src: int):
    """Concatenate every rank's 1-D tensor `t` (rank r holds sizes[r]
    elements) on `src`, in rank order; None elsewhere."""
    import torch

    dist = _dist()
    me = dist.get_rank()
    if me != src:
        if sizes[me]:
            _send(t[: sizes[me]].contiguous(), src)
        return None
    parts = []
    for r, n in enumerate(sizes):
        if r == me:
            parts.append(t[:n])
        elif n:
            buf = torch.empty(n, dtype=t.dtype, device=t.device)
            _recv(buf, r)
            parts.append(buf)
    return torch.cat(parts) if parts else t[:0]


def run_distributed_device(stream, config, upper_triangle_only: bool = False, src: int = 0):
    """run_parallel with the data path on the GPUs: rank
    `src` moves the stream to its GPU and broadcasts the arrays once (NCCL
    over NVLink; device to device), every rank counts the buckets of its
    contiguous block of worker intervals (the own-bucket layout for pair
    streams, the bucket-major partitions for real streams) and finalises
    their summaries -- each bucket lives on one rank, so the per-bucket
    top-l of the bounded regime is final there -- and the disjoint results
    are gathered to `src` as device arrays (point-to-point), with per-bucket
    loads, distinct counts, Count-Sketch cells and summary minima summed
    (each is non-zero only on its bucket's rank). `src` returns a device-
    backed (SketchState, LoadReport) equal to crop.run's; input_pair_total
    is 0 after a merge, as in the reference (engine.py:531)."""
    import torch

    from . import kernels
    from .engine import (LoadReport, SketchState, _check_positive_terms, _compute, _DeviceResult,
                         _Prepared, _worker_rows, prepare)
    from .errors import CropError, InputError

    dist = _dist()
    me, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", torch.cuda.current_device())
    meta = torch.zeros(9, dtype=torch.int64, device=dev)
    prep, failure = None, None
    if me == src:
        try:
            prep = prepare(stream)
            _check_positive_terms(prep, upper_triangle_only)
        except CropError as exc:  # every rank must leave the broadcast
            failure = exc
        if failure is None:
            d = prep.device
            if prep.kind == "pairs":
                meta[:8] = torch.tensor([0, prep.n_rows, prep.n_cols, prep.n_items, d.n_tx + 1, d.nnz, 0, 0])
            else:
                meta[:8] = torch.tensor([1, prep.n_rows, prep.n_cols, prep.n_items, d.n_products + 1,
                                         int(d.a_idx.numel()), int(d.b_idx.numel()), 0])
        else:
            meta[8] = 1
    _coll(dist.broadcast, meta, src)
    kind, n_rows, n_cols, n_items, n_ptr, nnz_a, nnz_b, _, err = (int(v) for v in meta.tolist())
    if err:
        if failure is not None:
            raise failure
        raise InputError(f"rank {src} rejected the stream")
    if kind == 0:
        if me == src:
            arrays = [prep.device.offsets, prep.device.items]
        else:
            arrays = [torch.empty(n_ptr, dtype=torch.int64, device=dev),
                      torch.empty(nnz_a, dtype=torch.int32, device=dev)]
        for t in arrays:
            _coll(dist.broadcast, t, src)
        if me != src:
            dtx = kernels.DeviceTransactions(arrays[0], arrays[1], n_items)
            prep = _Prepared("pairs", dtx, n_rows, n_cols, n_items, 0, None)
    else:
        if me == src:
            d = prep.device
            arrays = [d.a_ptr, d.a_idx, d.a_val, d.b_ptr, d.b_idx, d.b_val]
        else:
            arrays = [torch.empty(n_ptr, dtype=torch.int64, device=dev),
                      torch.empty(nnz_a, dtype=torch.int32, device=dev),
                      torch.empty(nnz_a, dtype=torch.float64, device=dev),
                      torch.empty(n_ptr, dtype=torch.int64, device=dev),
                      torch.empty(nnz_b, dtype=torch.int32, device=dev),
                      torch.empty(nnz_b, dtype=torch.float64, device=dev)]
        for t in arrays:
            _coll(dist.broadcast, t, src)
        if me != src:
            ds = kernels.DeviceOuterStream(*arrays, n_rows, n_cols)
            prep = _Prepared("outer", ds, n_rows, n_cols, n_items, 0, None)
    kappa = config.kappa
    asg = config.assignments()
    lo, hi = rank_workers(config.workers, me, world)  # hi > lo: workers >= world
    result, hashers = _compute(prep, config, upper_triangle_only, asg[lo].start, asg[hi - 1].stop)
    result.finalize_summaries()
    inst = result.instances[0]
    e = result.entries
    integer = result.integer
    # per-bucket facts, non-zero only on the bucket's rank: summed
    facts = torch.tensor(np.stack([inst.loads.astype(np.float64), inst.distinct.astype(np.float64),
                                   inst.cs.astype(np.float64) if inst.cs is not None else np.zeros(kappa),
                                   inst.bucket_min.astype(np.float64)]), dtype=torch.float64, device=dev)
    _coll(dist.all_reduce, facts)
    sizes_t = torch.zeros(world, dtype=torch.int64, device=dev)
    sizes_t[me] = e.n
    _coll(dist.all_reduce, sizes_t)
    sizes = [int(v) for v in sizes_t.tolist()]
    rec = inst.recorded
    if rec is None:
        rec = torch.ones(e.n, dtype=torch.bool, device=dev)
    cols = [e.row[: e.n], e.col[: e.n], rec[: e.n].to(torch.uint8)]
    cols += [e.count[: e.n]] if integer else [e.value[: e.n], e.bucket[: e.n]]
    got = [_gather_cat(c.contiguous(), sizes, src) for c in cols]
    if me != src:
        return None, None
    n = sum(sizes)
    if integer:
        row, col, rmask, cnt = got
        ent = kernels.DeviceEntries(row, col, cnt, None, n, 0)
    else:
        row, col, rmask, val, buck = got
        ent = kernels.DeviceEntries(row, col, None, val, n, 0, bucket=buck)
    f = facts.cpu().numpy()
    inst.loads = f[0].astype(np.int64)
    inst.distinct = f[1].astype(np.int64)
    inst.cs = f[2] if inst.cs is not None else None
    inst.bucket_min = f[3]
    inst.bucket_weight = None
    rmask = rmask.to(torch.bool)
    inst.recorded = None if bool(rmask.all().item()) else rmask
    merged = _DeviceResult(ent, integer, [inst], config.ss_capacity, kappa)
    state = SketchState._from_device(config, n_rows, n_cols, upper_triangle_only, merged)
    report = LoadReport(kappa=kappa, workers=config.workers, rows=[_worker_rows(inst.loads, asg)],
                        input_pair_total=0, assignments=[(a.start, a.stop) for a in asg])
    return state, report


def _coll(op, t, *args, **kw):
    """Run a collective on `t` with the process group's device: NCCL takes the
    CUDA tensor as is; gloo (CPU tests, several processes sharing one GPU)
    goes through a host copy, written back for in-place collectives."""
    dist = _dist()
    if dist.get_backend() == "nccl" or t.device.type == "cpu":
        return op(t, *args, **kw)
    h = t.cpu()
    r = op(h, *args, **kw)
    t.copy_(h)
    return r


def top_entries_distributed(stream, config, k: int, upper_triangle_only: bool = True,
                            src: int = 0):
    """Device path of a multi-GPU top-k mine (the benchmark's public call):
    SketchState.top_entries(k) of crop.run over all GPUs (engine.py:162-172).

    Rank `src` moves the stream to its GPU and broadcasts the CSR arrays once
    (NCCL over NVLink); each rank counts the buckets of its block of worker
    intervals only (crop_pairs with an interval filter), applies the bounded
    regime's per-bucket top-l summaries to its own buckets (each bucket lives
    on exactly one rank), and picks its local top-k; per-bucket loads and
    Count-Sketch cells are all-reduced and the k*G candidates gathered to
    `src`, which merges them. Returns (top entries, LoadReport) on `src`,
    (None, None) elsewhere. 0/1 self-join (mining) streams, one instance
    (an entry's buckets in several instances live on different ranks)."""
    import torch

    from . import kernels
    from .engine import LoadReport, TopEntry, _worker_rows, prepare
    from .errors import ConfigError
    from .hashing import HashConfig, make_hashes
    from .sparse import Entry

    if config.instances != 1:
        raise ConfigError("top_entries_distributed handles instances == 1 (use run_parallel)")
    if k < 0:
        raise ConfigError(f"k must be >= 0, got {k}")
    dist = _dist()
    me, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", torch.cuda.current_device())
    if me == src:
        prep = prepare(stream)
        if prep.kind != "pairs":
            raise ConfigError("top_entries_distributed handles 0/1 self-join streams")
        dtx = prep.device
        meta = torch.tensor([dtx.n_tx, dtx.nnz, dtx.n_items, prep.n_rows, prep.pair_total],
                            dtype=torch.int64, device=dev)
    else:
        meta = torch.zeros(5, dtype=torch.int64, device=dev)
    _coll(dist.broadcast, meta, src)
    n_tx, nnz, n_items, dim, pair_total = (int(v) for v in meta.tolist())
    if me != src:
        dtx = kernels.DeviceTransactions(torch.empty(n_tx + 1, dtype=torch.int64, device=dev),
                                         torch.empty(nnz, dtype=torch.int32, device=dev), n_items)
    _coll(dist.broadcast, dtx.offsets, src)
    _coll(dist.broadcast, dtx.items, src)
    kappa = config.kappa
    lo, hi = rank_workers(config.workers, me, world)
    asg = config.assignments()
    h = make_hashes(HashConfig(kappa, config.instance_seeds()[0]))
    tab = kernels.hash_tables(h, n_items)
    kk = max(k, 1)
    cand = torch.full((3, kk), -1, dtype=torch.int32, device=dev)
    loads = torch.zeros(kappa, dtype=torch.int64, device=dev)
    cells = torch.zeros(kappa, dtype=torch.int64, device=dev)
    if hi > lo and k > 0:
        ent = kernels.count_pairs(dtx, upper_triangle_only, kappa, asg[lo].start,
                                  asg[hi - 1].stop, *tab)
        signs = [h.sign_hash] if config.cs_enabled else None
        bl, distinct, cs = kernels.entry_bucket_stats(ent, [tab], kappa, n_items, signs)
        loads += bl[0]
        if cs is not None:
            cells += cs[0]
        count = None
        if int(distinct[0].max().item()) > config.ss_capacity:
            # bounded regime: only the per-bucket top-l records are candidates
            mask, _, _ = kernels.bucket_topk(ent, tab[0], tab[1], kappa, config.ss_capacity)
            count = torch.where(mask, ent.count[: ent.n], torch.zeros_like(ent.count[: ent.n]))
        idx = kernels.topk_indices(ent, k, count=count)
        if count is not None:
            idx = idx[count[idx] != 0]
        m = idx.shape[0]
        cand[0, :m], cand[1, :m], cand[2, :m] = ent.row[idx], ent.col[idx], ent.count[idx]
    elif hi > lo:
        ent = kernels.count_pairs(dtx, upper_triangle_only, kappa, asg[lo].start,
                                  asg[hi - 1].stop, *tab)
        bl, _, cs = kernels.entry_bucket_stats(ent, [tab], kappa, n_items,
                                               [h.sign_hash] if config.cs_enabled else None)
        loads += bl[0]
        if cs is not None:
            cells += cs[0]
    _coll(dist.all_reduce, loads)
    if config.cs_enabled:
        _coll(dist.all_reduce, cells)
    if dist.get_backend() == "nccl":
        gathered = [torch.empty_like(cand) for _ in range(world)] if me == src else None
        dist.gather(cand, gathered, dst=src)
    else:
        gathered = [torch.empty_like(cand).cpu() for _ in range(world)] if me == src else None
        dist.gather(cand.cpu(), gathered, dst=src)
    if me != src:
        return None, None
    if k == 0:
        top = []
    else:
        allc = torch.cat([g.cpu() for g in gathered], dim=1).numpy().view(np.uint32)
        allc = allc.astype(np.int64)
        keep = allc[2] != 0xFFFFFFFF
        r, c, w = allc[0][keep], allc[1][keep], allc[2][keep]
        order = np.lexsort((c, r, -w))[:k]
        cs_h = cells.cpu().numpy().astype(np.float64) if config.cs_enabled else None
        top = []
        for x in order:
            row, col, wt = int(r[x]), int(c[x]), float(w[x])
            est = float(cs_h[h.bucket_of(row, col)]) * h.sign_hash(row, col) \
                if cs_h is not None else None
            top.append(TopEntry(Entry(row, col), wt, wt, est))
    rows = [_worker_rows(loads.cpu().numpy(), asg)]
    report = LoadReport(kappa=kappa, workers=config.workers, rows=rows,
                        input_pair_total=pair_total,
                        assignments=[(a.start, a.stop) for a in asg])
    return top, report


def _a2a(out, inp, out_splits, in_splits):
    """all_to_all_single on the group's device (host copies under gloo)."""
    dist = _dist()
    if dist.get_backend() == "nccl" or inp.device.type == "cpu":
        dist.all_to_all_single(out, inp, out_splits, in_splits)
        return
    o = out.cpu()
    dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits)
    out.copy_(o)


def merge_bucket_summaries_distributed(ent, h_row, h_col, kappa: int, capacity: int):
    """Bounded-regime summaries of a job counted as tile shards across ranks
    (bench.py's N-GPU path): every rank holds exact counts of its tiles, and
    every bucket's pairs are spread over all ranks. Each rank keeps its own
    top-l candidates per bucket, sends them to the bucket's owner (rank r owns
    the buckets of split(kappa, world)[r], the reference's worker intervals,
    interval.py:37-45) with one all-to-all, and the owner selects the bucket's
    top-l among the union -- the same summary as one GPU counting everything
    (kernels.merge_bucket_summaries). Loads are all-reduced.

    Returns, for the caller's own buckets: (DeviceEntries of the received
    candidates, recorded mask, bucket_min int64[kappa] (zero outside the own
    interval), loads int64[kappa] (all buckets), distinct int64[kappa])."""
    import torch

    from . import kernels

    dist = _dist()
    me, world = dist.get_rank(), dist.get_world_size()
    dev = h_row.device
    n_items = int(h_row.shape[0])
    bl, dc, _ = kernels.entry_bucket_stats(ent, [(h_row, h_col)], kappa, n_items, None)
    loads, distinct = bl[0].clone(), dc[0].to(torch.int64)
    _coll(dist.all_reduce, loads)
    _coll(dist.all_reduce, distinct)
    n = ent.n
    row, col, cnt = ent.row[:n], ent.col[:n], ent.count[:n]
    if n and int(dc[0].max().item()) >= capacity:
        mask, _, _ = kernels.bucket_topk(ent, h_row, h_col, kappa, capacity)
        row, col, cnt = row[mask], col[mask], cnt[mask]
    b = kernels.entry_buckets(row, col, int(row.shape[0]), h_row, h_col, kappa).to(torch.int64)
    # the owner of bucket b is the rank whose split(kappa, world) interval holds it
    starts = torch.tensor([rank_workers(kappa, r, world)[0] for r in range(world)],
                          dtype=torch.int64, device=dev)
    owner = torch.bucketize(b, starts, right=True) - 1
    order = torch.argsort(owner, stable=True)
    row, col, cnt, owner = row[order], col[order], cnt[order], owner[order]
    send = torch.bincount(owner, minlength=world).to(torch.int64)
    recv = torch.empty_like(send)
    _a2a(recv, send, None, None)
    s_l, r_l = send.cpu().tolist(), recv.cpu().tolist()
    total = int(sum(r_l))
    packed = torch.stack([row, col, cnt])  # int32 [3, m]
    out = torch.empty((3, max(total, 1)), dtype=torch.int32, device=dev)
    for k in range(3):
        buf = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        _a2a(buf[:total], packed[k].contiguous(), r_l, s_l)
        out[k] = buf
    cand = kernels.DeviceEntries(out[0, :total].contiguous(), out[1, :total].contiguous(),
                                 out[2, :total].contiguous(), None, total, ent.total_terms)
    if total:
        mask, bmin, _ = kernels.bucket_topk(cand, h_row, h_col, kappa, capacity)
    else:
        mask = torch.zeros(0, dtype=torch.bool, device=dev)
        bmin = torch.zeros(kappa, dtype=torch.int64, device=dev)
    lo, hi = rank_workers(kappa, me, world)
    own = torch.zeros(kappa, dtype=torch.bool, device=dev)
    own[lo:hi] = True
    bmin = torch.where(own & (distinct >= capacity), bmin, torch.zeros_like(bmin))
    return cand, mask, bmin, loads, distinct
