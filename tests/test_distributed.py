"""Multi-process orchestration of the multi-GPU path, on CPU (gloo, world 2).

The per-rank compute is injected: the C oracle produces each rank's worker
payloads (as the GPU engine does on a B200), so these tests cover exactly
the host-side logic -- broadcast once, rank -> worker-block mapping, disjoint
payload gather, merge with tiling validation -- and check the merged state
against a single-process oracle run (K-invariance).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_1210_0461_b200 as crop
from paper_1210_0461_b200 import distributed, hashing


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def oracle_payloads(stream, config, w_lo, w_hi, upper):
    """Worker payloads (crop-partial/1) computed by the C oracle."""
    out = []
    asg = config.assignments()
    ost = oracle.Stream(stream.offsets, stream.items)
    for w in range(w_lo, w_hi):
        insts = []
        for seed in config.instance_seeds():
            h = crop.make_hashes(crop.HashConfig(config.kappa, seed))
            recs, load = oracle.run_worker(ost, h.coefficients(), config.kappa, config.workers, w,
                                           capacity=0, upper_only=upper, cs=config.cs_enabled)
            summaries = []
            for b in sorted(set(recs.bucket.tolist())):
                sel = recs.bucket == b
                lines = [f"capacity {config.ss_capacity}",
                         f"total_weight {float(recs.bucket_totals[b])!r}"]
                lines += [f"{r} {c} {n!r} 0.0" for r, c, n in
                          zip(recs.row[sel].tolist(), recs.col[sel].tolist(),
                              recs.count[sel].tolist())]
                summaries.append([int(b), lines])
            cells = None
            if config.cs_enabled:
                cells = [float(x) for x in recs.cs[asg[w].start:asg[w].stop]]
            insts.append({"seed": seed, "hashes": hashing.hasher_to_text(h, seed), "count": load,
                          "summaries": summaries, "cs_cells": cells})
        out.append({"format": "crop-partial/1", "worker": w, "start": asg[w].start,
                    "stop": asg[w].stop, "n_rows": stream.n_rows, "n_cols": stream.n_cols,
                    "upper_triangle_only": upper, "config": config.to_dict(),
                    "instances": insts})
    return out


def _state_records(state):
    res = []
    for inst in state.instances:
        rs = sorted((b, it[0], it[1], c) for b, s in inst.summaries.items()
                    for it, c, _ in s.records())
        res.append((rs, inst.sketch.cells if inst.sketch else None))
    return res


def _worker(rank, world, port, tx, cfg_dict, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        config = crop.EngineConfig(**cfg_dict)
        stream = crop.transactions_to_stream(tx) if rank == 0 else None
        state, report = distributed.run_distributed(stream, config, True, compute=oracle_payloads)
        # broadcast_arrays round trip of mixed dtypes
        arr = {"a": np.arange(7, dtype=np.uint32) * 3, "b": np.linspace(0, 1, 5),
               "c": np.array([2 ** 40, 5], dtype=np.int64)} if rank == 0 else None
        got = distributed.broadcast_arrays(arr)
        ok = (got["a"].tolist() == (np.arange(7) * 3).tolist() and got["b"].tolist() ==
              np.linspace(0, 1, 5).tolist() and got["c"].tolist() == [2 ** 40, 5])
        if rank == 0:
            q.put((_state_records(state), report.rows, ok))
        else:
            q.put(("peer", state is None and report is None, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("workers,kappa,instances", [(4, 4, 1), (3, 12, 3), (1, 5, 1)])
def test_run_distributed_world2_matches_single_process(golden, workers, kappa, instances):
    tx = golden["mining"][1]["transactions"]
    cfg = crop.EngineConfig(kappa=kappa, ss_capacity=2 ** 31, workers=workers, cs_enabled=True,
                            instances=instances, seed=3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tx, cfg.to_dict(), q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    main = next(r for r in results if r[0] != "peer")
    peer = next(r for r in results if r[0] == "peer")
    assert peer[1] and peer[2] and main[2]
    # single-process reference: all workers through the same oracle payloads
    stream = crop.transactions_to_stream(tx)
    single, rep = crop.merge_partials(oracle_payloads(stream, cfg, 0, cfg.workers, True))
    assert main[0] == _state_records(single)
    assert main[1] == rep.rows


def test_rank_worker_blocks_tile_all_workers():
    for workers in range(1, 20):
        for world in range(1, 9):
            blocks = [distributed.rank_workers(workers, r, world) for r in range(world)]
            covered = [w for lo, hi in blocks for w in range(lo, hi)]
            assert covered == list(range(workers))
