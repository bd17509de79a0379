"""The CLI retarget (cli.py) against the reference CLI's own outputs
(tests/golden: generate transactions, then mine with --exact-oracle)."""

import csv
import io
import json

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1210_0461_b200 import cli  # noqa: E402


def _csv(text):
    return list(csv.reader(io.StringIO(text)))


def test_generate_and_mine_match_reference_cli(golden, tmp_path):
    case = golden["cli"]
    gen = tmp_path / "gen"
    assert cli.main(["generate", "transactions", *case["generate_transactions"]["args"],
                     "--out", str(gen)]) == 0
    assert (gen / "transactions.fimi").read_text() == case["generate_transactions"]["fimi"]
    assert (gen / "pair_supports.csv").read_text() == case["generate_transactions"]["pair_supports"]
    out = tmp_path / "mine"
    assert cli.main(["mine", "--fimi", str(gen / "transactions.fimi"), "--out", str(out),
                     *case["mine"]["args"]]) == 0
    want = case["mine"]["outputs"]
    assert _csv((out / "topk.csv").read_text()) == _csv(want["topk.csv"])
    assert json.loads((out / "load_report.json").read_text()) == json.loads(want["load_report.json"])
    assert _csv((out / "bound_ratios.csv").read_text()) == _csv(want["bound_ratios.csv"])
    got_state = json.loads((out / "state.json").read_text())
    want_state = json.loads(want["state.json"])
    for g, w in zip(got_state["instances"], want_state["instances"]):
        assert g["hashes"] == w["hashes"] and g["cs"] == w["cs"]
        assert {b: (lines[:2], sorted(lines[2:])) for b, lines in g["summaries"]} == \
            {b: (lines[:2], sorted(lines[2:])) for b, lines in w["summaries"]}
    manifest = json.loads((out / "manifest.json").read_text())
    assert manifest["load"]["max_avg_ratio"] == json.loads(want["load_report.json"])["max_avg_ratio"]


def test_bench_reports_gpu_rows(golden, tmp_path):
    fimi = tmp_path / "t.fimi"
    fimi.write_text(golden["cli"]["generate_transactions"]["fimi"])
    out = tmp_path / "bench"
    assert cli.main(["bench", "--fimi", str(fimi), "--kappa", "8", "--workers-list", "1,4096",
                     "--out", str(out)]) == 0
    rows = json.loads((out / "manifest.json").read_text())["rows"]
    assert rows[0]["gpus"] == 1 and rows[0]["terms_per_second"] > 0
    assert 0 < rows[0]["hbm_roofline_fraction"] < 1
    assert rows[1]["gpus"] == 4096 and "unavailable" in rows[1]
