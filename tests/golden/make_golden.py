"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package under the alias `crop_ref` (so it cannot
collide with anything in this repo), feeds it small seeded inputs, and writes
its outputs to tests/golden/*.json. Those fixtures pin both the C oracle
(tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_parity.py).
Nothing at test time reads /root/reference.
"""

import importlib.util
import json
import os
import random
import sys

REF_SRC = "/root/reference/pkg/src/crop"
HERE = os.path.dirname(os.path.abspath(__file__))


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "crop_ref", os.path.join(REF_SRC, "__init__.py"), submodule_search_locations=[REF_SRC])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["crop_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def gen_transactions(rng, n_tx, n_items, max_len, skew=1.1):
    """Small skewed transactions (ids sorted, distinct)."""
    weights = [1.0 / (r + 1) ** skew for r in range(n_items)]
    out = []
    for _ in range(n_tx):
        size = rng.randint(0, max_len)
        items = set()
        while len(items) < min(size, n_items):
            items.add(rng.choices(range(n_items), weights)[0])
        out.append(sorted(items))
    return out


def coeffs_of(h):
    return [h.row_hash.mul, h.row_hash.add, h.col_hash.mul, h.col_hash.add, h.sign_hash.mul,
            h.sign_hash.add]


def state_records(state):
    inst_out = []
    for inst in state.instances:
        recs = []
        for bucket in sorted(inst.summaries):
            s = inst.summaries[bucket]
            for item, count, over in s.records():
                recs.append([bucket, item[0], item[1], count, over])
        totals = {str(b): inst.summaries[b].total_weight for b in sorted(inst.summaries)}
        inst_out.append({
            "seed": inst.seed,
            "coeffs": coeffs_of(inst.hasher),
            "records": recs,
            "bucket_totals": totals,
            "cs": None if inst.sketch is None else list(inst.sketch.cells),
        })
    return inst_out


def main():
    crop = load_reference()
    rng = random.Random(20121002)
    golden = {}

    # -- hashing: coefficients, per-item tables, signs, seeds --------------------
    hashes = []
    for kappa, seed in [(16, 42), (4, 0), (8, 1), (1184, 7), (1, 3), (65536, 123456789),
                        (3, 2 ** 63 + 5)]:
        h = crop.make_hashes(crop.HashConfig(kappa, seed))
        idx = list(range(64)) + [1000, 65535, 65536, 10 ** 6, 2 ** 31, 2 ** 32 - 1]
        signs = [[i, j, h.sign_hash(i, j)] for i, j in [(1, 2), (0, 0), (5, 3), (2 ** 32 - 1, 7),
                                                         (123456, 2 ** 32 - 1), (17, 17)]]
        hashes.append({"kappa": kappa, "seed": seed, "coeffs": coeffs_of(h), "indices": idx,
                       "h_row": h.row_hash.values(idx), "h_col": h.col_hash.values(idx),
                       "signs": signs, "text": crop.hashing.hasher_to_text(h, seed)})
    golden["hashes"] = hashes
    golden["derive_seed"] = [[m, lab, crop.derive_seed(m, lab)] for m, lab in
                             [(0, "instance:0"), (0, "instance:1"), (7, "instance:4"),
                              (2 ** 40, "instance:0"), (1, "data")]]
    golden["instance_seeds"] = [[s, t, crop.EngineConfig(kappa=8, ss_capacity=4, seed=s,
                                                         instances=t).instance_seeds()]
                                for s, t in [(0, 1), (0, 3), (5, 5)]]

    # -- bucket_sort_indices, both branches ------------------------------------
    bsort = []
    for kappa, n, comb in [(8, 12, None), (1000, 6, None), (64, 30, 100), (5, 0, None)]:
        h = crop.make_hashes(crop.HashConfig(kappa, kappa + n))
        idx = sorted(rng.sample(range(500), n))
        vals = [rng.choice([1.0, -2.5, 0.5, 3.0]) for _ in idx]
        v = crop.SparseVector(500, idx, vals)
        out = crop.bucket_sort_indices(v, h.row_hash, comb)
        bsort.append({"kappa": kappa, "coeffs": coeffs_of(h), "indices": idx, "values": vals,
                      "combined": comb, "hashes": out.hashes, "sorted_indices": out.indices,
                      "sorted_values": out.values})
    golden["bucket_sort"] = bsort

    # -- pair mining streams through run / measure_loads ----------------------
    mining = []
    cases = [
        # n_tx, n_items, max_len, kappa, workers, capacity, instances, seed
        (300, 40, 12, 4, 4, 2 ** 31, 1, 0),
        (400, 120, 20, 8, 2, 2 ** 31, 3, 5),
        (250, 60, 15, 16, 4, 3, 1, 11),     # Space-Saving regime (evictions)
        (200, 30, 10, 1, 1, 5, 1, 2),       # kappa = 1, tiny summaries
        (150, 500, 25, 64, 8, 2 ** 31, 1, 9),
    ]
    for n_tx, n_items, max_len, kappa, workers, cap, inst, seed in cases:
        tx = gen_transactions(rng, n_tx, n_items, max_len)
        stream = crop.transactions_to_stream(tx)
        cfg = crop.EngineConfig(kappa=kappa, ss_capacity=cap, workers=workers, cs_enabled=True,
                                instances=inst, seed=seed)
        state, report = crop.run(stream, cfg, upper_triangle_only=True)
        loads_upper = crop.measure_loads(stream, cfg, upper_triangle_only=True)
        loads_full = crop.measure_loads(stream, cfg, upper_triangle_only=False)
        top = [[t.entry.row, t.entry.col, t.lower, t.upper, t.estimate]
               for t in state.top_entries(25)]
        queries = []
        for i, j in [(0, 1), (1, 2), (0, n_items - 1), (3, 3), (2, 0)]:
            lo, up, est = state.query((i, j))
            queries.append([i, j, lo, up, est])
        mining.append({
            "transactions": tx, "dim": stream.n_rows,
            "config": cfg.to_dict(), "instances": state_records(state),
            "rows": report.rows, "input_pair_total": report.input_pair_total,
            "assignments": report.assignments, "max_avg_ratio": report.max_avg_ratio(),
            "loads_upper": loads_upper.rows, "loads_full": loads_full.rows,
            "pair_total_full": loads_full.input_pair_total,
            "top25": top, "queries": queries,
            "supports": sorted([list(k) + [v] for k, v in crop.exact_pair_supports(tx).items()]),
        })
    golden["mining"] = mining

    # -- full (non-triangle) self-join run --------------------------------------
    tx = gen_transactions(rng, 120, 30, 8)
    stream = crop.transactions_to_stream(tx)
    cfg = crop.EngineConfig(kappa=6, ss_capacity=2 ** 31, workers=3, cs_enabled=True, seed=4)
    state, report = crop.run(stream, cfg, upper_triangle_only=False)
    golden["selfjoin_full"] = {"transactions": tx, "config": cfg.to_dict(),
                               "instances": state_records(state), "rows": report.rows}

    # -- general real-valued streams: exact_product and partition enumeration ---
    general = []
    for n_k, n_dim, max_nnz, kappa, workers, seed in [(60, 50, 8, 4, 2, 1), (40, 300, 20, 12, 4, 2),
                                                      (30, 20, 6, 1, 1, 3)]:
        pairs = []
        for _ in range(n_k):
            ai = sorted(rng.sample(range(n_dim), rng.randint(0, max_nnz)))
            bi = sorted(rng.sample(range(n_dim), rng.randint(0, max_nnz)))
            av = [rng.choice([-1.5, 2.0, 0.25, 1.0, -3.0, 0.1]) for _ in ai]
            bv = [rng.choice([1.0, -0.5, 4.0, 0.3, 7.0]) for _ in bi]
            pairs.append((crop.SparseVector(n_dim, ai, av), crop.SparseVector(n_dim, bi, bv)))
        stream = crop.OuterProductStream.from_pairs(n_dim, n_dim, pairs)
        h = crop.make_hashes(crop.HashConfig(kappa, seed))
        parts = []
        for asg in crop.WorkerAssignment.split(kappa, workers):
            acc = {}
            count = 0
            for a, b in stream:
                count += crop.count_interval(a, b, h.row_hash, h.col_hash, asg)
                for e, v in crop.enumerate_interval(a, b, h.row_hash, h.col_hash, asg):
                    acc[tuple(e)] = acc.get(tuple(e), 0.0) + v
            parts.append({"start": asg.start, "stop": asg.stop, "count": count,
                          "entries": sorted([list(k) + [v] for k, v in acc.items()])})
        exact = crop.exact_product(stream)
        exact_upper = crop.exact_product(stream, upper_only=True)
        general.append({
            "n_dim": n_dim, "kappa": kappa, "workers": workers, "seed": seed,
            "coeffs": coeffs_of(h),
            "a": [[list(a.indices), list(a.values)] for a, _ in pairs],
            "b": [[list(b.indices), list(b.values)] for _, b in pairs],
            "partitions": parts,
            "exact": sorted([list(k) + [v] for k, v in exact.items()]),
            "exact_upper": sorted([list(k) + [v] for k, v in exact_upper.items()]),
        })
    golden["general"] = general

    # -- Space-Saving unit behaviour ------------------------------
    ss_cases = []
    for cap, seq in [(1, [["a", 1.0], ["b", 1.0], ["a", 1.0]]),
                     (2, [["x", 2.0], ["y", 1.0], ["z", 1.0], ["y", 3.0], ["w", 0.5]]),
                     (3, [[str(rng.randint(0, 6)), float(rng.randint(1, 4))] for _ in range(40)])]:
        s = crop.SpaceSavingSummary(cap)
        for item, w in seq:
            s.update(item, w)
        ss_cases.append({"capacity": cap, "updates": seq,
                         "records": [[it, c, o] for it, c, o in s.records()],
                         "total": s.total_weight, "min": s.min_count(),
                         "queries": {q: list(s.query(q)) for q in ["a", "b", "x", "y", "z", "w",
                                                                    "0", "1", "2", "9"]}})
    golden["spacesaving"] = ss_cases

    # ---- round 2 additions (appended so every fixture above is unchanged) ----
    # LoadReport.max_avg_ratio rounding (engine.py:207-216) on random rows
    ratio_rows = []
    for _ in range(400):
        width = rng.randint(1, 12)
        rows = [[rng.randint(0, 10 ** rng.randint(1, 9)) for _ in range(width)]
                for _ in range(rng.randint(1, 3))]
        rep = crop.LoadReport(kappa=width, workers=width, rows=rows, input_pair_total=0)
        ratio_rows.append([rows, rep.max_avg_ratio()])
    golden["max_avg_ratio"] = ratio_rows

    # per-product worker loads (engine.py:250-251,287-288; measure_loads :305-349)
    per_product = []
    for n_tx, n_items, max_len, kappa, workers, seed, upper in [(120, 50, 14, 8, 3, 1, True),
                                                                (90, 200, 30, 64, 5, 2, False)]:
        tx = gen_transactions(rng, n_tx, n_items, max_len)
        stream = crop.transactions_to_stream(tx)
        cfg = crop.EngineConfig(kappa=kappa, ss_capacity=2 ** 31, workers=workers,
                                cs_enabled=False, seed=seed)
        _, rep = crop.run(stream, cfg, upper_triangle_only=upper, record_per_product=True)
        ml = crop.measure_loads(stream, cfg, upper_triangle_only=upper, record_per_product=True)
        per_product.append({"transactions": tx, "config": cfg.to_dict(), "upper": upper,
                            "run": [list(x[:2]) + [list(x[2])] for x in rep.per_product],
                            "measure": [list(x[:2]) + [list(x[2])] for x in ml.per_product]})
    golden["per_product"] = per_product

    # run_worker payloads (engine.py:396-455), exact regime, 3 instances + Count-Sketch
    tx = gen_transactions(rng, 200, 80, 16)
    stream = crop.transactions_to_stream(tx)
    cfg = crop.EngineConfig(kappa=12, ss_capacity=2 ** 31, workers=4, cs_enabled=True,
                            instances=3, seed=21)
    golden["run_worker"] = {"transactions": tx, "config": cfg.to_dict(),
                            "payloads": [crop.run_worker(stream, cfg, w, upper_triangle_only=True)
                                         for w in range(cfg.workers)]}

    # Zipf generators (oracle.py:74-185)
    zs = []
    for scale, skew, distinct, dim, outer, seed in [(100.0, 1.2, 30, 12, None, 1),
                                                     (5.0, 0.8, 20, 9, 20, 2),
                                                     (1.0, 1.5, 12, 6, 17, 3)]:
        s = crop.gen_zipf_stream(crop.ZipfModel(scale, skew, distinct), dim, outer, seed)
        zs.append({"args": [scale, skew, distinct, dim, outer, seed],
                   "products": [[list(a.indices), list(a.values), list(b.indices), list(b.values)]
                                for a, b in s]})
    zt = []
    for n_items, n_tx, skew, seed, mean in [(200, 40, 1.1, 5, 10), (30, 25, 0.7, 9, 4),
                                            (5, 10, 2.0, 0, 8)]:
        zt.append({"args": [n_items, n_tx, skew, seed, mean],
                   "transactions": [list(t) for t in
                                    crop.gen_zipf_transactions(n_items, n_tx, skew, seed, mean)]})
    golden["zipf"] = {"streams": zs, "transactions": zt}

    # triple files (sparse.py:173-254): valid files through load_column_row_streams
    # and malformed ones with the reference's ParseError line numbers
    import tempfile

    def triple_text(vectors, n_rows, n_cols, blank_every=0, crlf=False, shuffle_within=False):
        lines = [f"{n_rows} {n_cols} {len(vectors)}"]
        for k, vec in enumerate(vectors):
            pairs = list(vec)
            if shuffle_within:
                rng.shuffle(pairs)
            for idx, val in pairs:
                lines.append(f"{k} {idx} {val!r}")
                if blank_every and rng.random() < 1.0 / blank_every:
                    lines.append("   ")
        nl = "\r\n" if crlf else "\n"
        return nl.join(lines) + nl

    def rand_vectors(n_vec, dim, max_nnz, zero_prob=0.0):
        out = []
        for _ in range(n_vec):
            idx = sorted(rng.sample(range(dim), rng.randint(0, max_nnz)))
            vals = [0.0 if rng.random() < zero_prob else
                    rng.choice([1.5, -2.25, 3e-7, 1e22, -0.125, 7.0, 2.5e-300]) *
                    (1 + rng.randint(0, 999) / 1000) for _ in idx]
            out.append(list(zip(idx, vals)))
        return out

    triples = []
    with tempfile.TemporaryDirectory() as td:
        for n_vec, dim, max_nnz, kw in [(40, 60, 8, {}), (25, 30, 5, {"blank_every": 4}),
                                        (30, 500, 12, {"crlf": True, "shuffle_within": True}),
                                        (10, 20, 6, {"zero": 0.3})]:
            zero = kw.pop("zero", 0.0)
            va = rand_vectors(n_vec, dim, max_nnz, zero)
            vb = rand_vectors(n_vec, dim, max_nnz, zero)
            ta = triple_text(va, dim, dim, **kw)
            tb = triple_text(vb, dim, dim, **kw)
            pa, pb = os.path.join(td, "a.t"), os.path.join(td, "b.t")
            with open(pa, "w", newline="") as fh:
                fh.write(ta)
            with open(pb, "w", newline="") as fh:
                fh.write(tb)
            s = crop.load_column_row_streams(pa, pb)
            triples.append({"a": ta, "b": tb, "ok": True,
                            "zeros": s.zero_values_dropped,
                            "products": [[list(a.indices), list(a.values), list(b.indices),
                                          list(b.values)] for a, b in s]})
        bad_cases = [
            "3 3\n",                                   # header fields
            "3 3 2\n0 1 1.0\n1 2 x\n",                 # malformed value
            "3 3 2\n1 1 1.0\n0 2 2.0\n",               # unsorted k
            "3 3 2\n0 1 1.0\n2 2 2.0\n",               # k out of range
            "3 3 2\n0 -1 1.0\n",                       # negative index
            "3 3 2\n0 1 nan\n",                        # NaN
            "3 3 2\n0 1 1.0 5\n",                      # four fields
            "3 3 2\n0 1 2.0\n0 1 3.0\n",               # duplicate index (line 0)
            "",                                        # missing header
            "3 3 2\n0 1 1_000.5\n1 2 +2\n",            # unusual but valid spelling
            "3 3 2\n\n0 1 inf\n1 0 -0.0\n",            # inf kept, -0.0 dropped
        ]
        for text in bad_cases:
            pa = os.path.join(td, "bad.t")
            with open(pa, "w", newline="") as fh:
                fh.write(text)
            try:
                r, c, groups, zeros = crop.sparse.read_triple_file(pa)
                triples.append({"a": text, "ok": True, "side_only": True, "header": [r, c],
                                "groups": [[list(p) for p in g] for g in groups],
                                "zeros": zeros})
            except crop.ParseError as exc:
                triples.append({"a": text, "ok": False, "side_only": True,
                                "line_no": exc.line_no,
                                "message": str(exc).split(": ", 1)[1]})
    golden["triples"] = triples

    # the reference CLI (cli.py): mine and generate outputs on small inputs
    from crop_ref import cli as ref_cli

    cli_cases = {}
    with tempfile.TemporaryDirectory() as td:
        gen_dir = os.path.join(td, "gen")
        assert ref_cli.main(["generate", "transactions", "--items", "120", "--count", "300",
                             "--skew", "1.1", "--mean-size", "9", "--seed", "4",
                             "--out", gen_dir]) == 0
        with open(os.path.join(gen_dir, "transactions.fimi")) as fh:
            fimi = fh.read()
        with open(os.path.join(gen_dir, "pair_supports.csv")) as fh:
            supports_csv = fh.read()
        cli_cases["generate_transactions"] = {
            "args": ["--items", "120", "--count", "300", "--skew", "1.1", "--mean-size", "9",
                     "--seed", "4"], "fimi": fimi, "pair_supports": supports_csv}
        mine_dir = os.path.join(td, "mine")
        margs = ["--kappa", "8", "--workers", "4", "--ss-capacity", "1000000", "--seed", "3",
                 "--top", "30", "--exact-oracle"]
        assert ref_cli.main(["mine", "--fimi", os.path.join(gen_dir, "transactions.fimi"),
                             "--out", mine_dir] + margs) == 0
        outs = {}
        for name in ("topk.csv", "load_report.json", "bound_ratios.csv", "state.json"):
            with open(os.path.join(mine_dir, name)) as fh:
                outs[name] = fh.read()
        cli_cases["mine"] = {"args": margs, "outputs": outs}
        rc_bad = ref_cli.main(["mine", "--fimi", os.path.join(td, "missing.fimi"), "--kappa", "4",
                               "--out", os.path.join(td, "x")])
        rc_cfg = ref_cli.main(["mine", "--fimi", os.path.join(gen_dir, "transactions.fimi"),
                               "--kappa", "4", "--workers", "9", "--out", os.path.join(td, "y")])
        cli_cases["exit_codes"] = {"missing_input": rc_bad, "bad_workers": rc_cfg}
    golden["cli"] = cli_cases

    with open(os.path.join(HERE, "reference_golden.json"), "w") as fh:
        json.dump(golden, fh, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
