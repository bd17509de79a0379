"""Multi-rank paths with the real GPU compute: two gloo processes sharing one
GPU (the ranks never wait on each other's kernels -- collectives run on the
host), compared with the single-process crop.run on the same stream.

Covers distributed.run_distributed (one instance: the device path with device
broadcast, per-rank bucket intervals and point-to-point gather of the device
results; several instances: worker_payloads, pickled crop-partial/1 gather,
merge_partials) and distributed.top_entries_distributed
(bucket-interval counting per rank, loads / Count-Sketch all-reduce, top-k
gather), including the bounded Space-Saving regime.
"""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import distributed  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _records(state):
    res = []
    for inst in state.instances:
        rs = sorted((b, it[0], it[1], c, o) for b, s in inst.summaries.items()
                    for it, c, o in s.records())
        res.append((rs, inst.sketch.cells if inst.sketch else None))
    return res


def _top(top):
    return [(t.entry.row, t.entry.col, t.lower, t.upper, t.estimate) for t in top]


def _worker(rank, world, port, tx, cfg_dict, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        config = crop.EngineConfig(**cfg_dict)
        stream = crop.transactions_to_stream(tx) if rank == 0 else None
        state, report = distributed.run_distributed(stream, config, True)
        out = {}
        if rank == 0:
            out["records"] = _records(state)
            out["rows"] = report.rows
        if config.instances == 1:
            top, rep2 = distributed.top_entries_distributed(stream, config, k, True)
            if rank == 0:
                out["top"] = _top(top)
                out["rows2"] = rep2.rows
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _spawn(tx, cfg, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tx, cfg.to_dict(), k, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res[0]


@pytest.mark.parametrize("workers,kappa,instances,cap,cs", [
    (4, 8, 1, 2 ** 31, True), (3, 12, 3, 2 ** 31, True), (4, 4, 1, 3, False),
    (5, 1184, 1, 2 ** 31, False)])
def test_distributed_gpu_matches_single_process(golden, workers, kappa, instances, cap, cs):
    tx = golden["mining"][1]["transactions"] + golden["mining"][4]["transactions"]
    cfg = crop.EngineConfig(kappa=kappa, ss_capacity=cap, workers=workers, cs_enabled=cs,
                            instances=instances, seed=7)
    got = _spawn(tx, cfg, 40)
    stream = crop.transactions_to_stream(tx)
    state, report = crop.run(stream, cfg, upper_triangle_only=True)
    assert got["rows"] == report.rows
    want = _records(state)
    if cap >= 2 ** 31:
        assert got["records"] == want
    else:
        # bounded regime: the merged summaries hold the same per-bucket top-l
        # records as the single-process run (both derive them from exact counts)
        assert [r for r, _ in got["records"]] == [r for r, _ in want]
    if instances == 1:
        assert got["top"] == _top(state.top_entries(40))
        assert got["rows2"] == report.rows


def _merge_worker(rank, world, port, n_tx, cap, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1210_0461_b200 import kernels, workloads

        cfg = workloads.CONFIGS["c3"]
        dtx = workloads.generate_pairs_workload(cfg, n_tx=n_tx)
        h = crop.make_hashes(crop.HashConfig(cfg.kappa, crop.derive_seed(0, "instance:0")))
        tab = kernels.hash_tables(h, cfg.n_items)
        ent = kernels.count_pairs_shard(dtx, True, None, keep=tab, shard=(rank, world))
        cand, mask, bmin, loads, distinct = distributed.merge_bucket_summaries_distributed(
            ent, tab[0], tab[1], cfg.kappa, cap)
        rec = torch.stack([cand.row[mask], cand.col[mask]]).cpu().numpy().view("uint32")
        q.put((rank, rec.astype("int64").tolist(), bmin.cpu().tolist(), loads.cpu().tolist()))
    finally:
        dist.destroy_process_group()


def test_tile_shard_summaries_merge_across_ranks():
    """Bounded-regime summaries of 3 tile-shard ranks merged with the
    bucket-owner all-to-all equal the single-GPU summaries (c3 prefix)."""
    import numpy as np

    from paper_1210_0461_b200 import kernels, workloads

    n_tx, cap, world = 20_000, 256, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_merge_worker, args=(r, world, port, n_tx, cap, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (rec, bmin, loads)) for r, rec, bmin, loads in
               (q.get(timeout=600) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = workloads.CONFIGS["c3"]
    dtx = workloads.generate_pairs_workload(cfg, n_tx=n_tx)
    config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=cap, workers=world, seed=0,
                               cs_enabled=False)
    state, _ = crop.run(dtx, config, upper_triangle_only=True)
    d = state.device_result
    e, inst = d.entries, d.instances[0]
    m = inst.recorded
    whole = np.stack([kernels.u32_to_numpy(e.row[: e.n][m]), kernels.u32_to_numpy(e.col[: e.n][m])])
    whole_keys = set(map(tuple, whole.T.astype(np.int64).tolist()))
    got_keys = set()
    bmin = np.zeros(cfg.kappa, np.int64)
    for r in range(world):
        rec, bm, loads = res[r]
        got_keys |= set(zip(rec[0], rec[1]))
        bmin += np.array(bm)
        assert loads == inst.loads.astype(np.int64).tolist()
    assert got_keys == whole_keys
    assert bmin.tolist() == inst.bucket_min.astype(np.int64).tolist()


def _outer_worker(rank, world, port, arrays, cfg_dict, upper, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        config = crop.EngineConfig(**cfg_dict)
        stream = crop.ColumnRowStream(*arrays) if rank == 0 else None
        state, report = distributed.run_distributed(stream, config, upper)
        out = {}
        if rank == 0:
            out["records"] = _records(state)
            out["rows"] = report.rows
            out["total"] = report.input_pair_total
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,workers,cap,upper", [(2, 4, 2 ** 31, False), (3, 6, 40, True)])
def test_device_run_distributed_real_stream(world, workers, cap, upper):
    """run_distributed's device path on a real-valued CSC/CSR stream (bucket-
    major partitions per rank, device broadcast and point-to-point gather):
    the merged summaries equal single-process crop.run's, in the exact and
    the bounded regime."""
    from paper_1210_0461_b200 import workloads

    cfg4 = workloads.CONFIGS["c4"]
    s = workloads.generate_product_workload(cfg4, n_products=3_000)
    pos = (s.a_ptr, s.a_idx, abs(s.a_val) + 0.5, s.b_ptr, s.b_idx, abs(s.b_val) + 0.5)
    arrays = (cfg4.n, cfg4.n) + pos
    cfg = crop.EngineConfig(kappa=24, ss_capacity=cap, workers=workers, cs_enabled=True, seed=5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_outer_worker, args=(r, world, port, arrays, cfg.to_dict(), upper, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = res[0]
    state, report = crop.run(crop.ColumnRowStream(*arrays), cfg, upper_triangle_only=upper)
    assert got["rows"] == report.rows
    assert got["total"] == 0
    want = _records(state)
    assert [r for r, _ in got["records"]] == [r for r, _ in want]
    np_cells_got, np_cells_want = got["records"][0][1], want[0][1]
    assert np_cells_got == pytest.approx(np_cells_want, rel=1e-12, abs=1e-9)
