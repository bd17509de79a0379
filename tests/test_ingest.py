"""Native FIMI ingestion against the reference-exact
Python reader: same CSR, same duplicate accounting, same errors (CPU only:
the reader is host code in libcrop_b200.so)."""

import numpy as np
import pytest

import paper_1210_0461_b200 as crop
from paper_1210_0461_b200 import mining, sparse


def _python_csr(path):
    rows = sparse.read_fimi(path)
    off, items = sparse._csr_from_lists(rows)
    return off, items.astype(np.uint32)


@pytest.mark.parametrize("text", [
    "3 1 2\n\n  5 5 7\t9\r\n+4 -0 04\n10\n",   # blank line, CRLF, signs, leading zeros
    "",                                         # empty file
    "\n\n   \n",                                # blank lines only
    "7",                                        # no final newline
    "1 2\r",                                    # CR at end of file
    "1 2\r3 4\n",                               # bare CR: a universal newline (Python reader)
    "1_000 2\n",                                # digit separator (Python int accepts it)
    "٣ 2\n",                               # non-ASCII digit (Python int accepts it)
    "2147483647 0\n",                           # ids >= 2^31 go to the Python reader
])
def test_native_reader_matches_reference_reader(tmp_path, text):
    p = tmp_path / "t.dat"
    p.write_text(text, encoding="utf-8")
    off, items, mx = sparse.read_fimi_csr(p)
    ro, ri = _python_csr(p)
    assert np.array_equal(off, ro) and np.array_equal(items, ri)
    assert mx == (int(ri.max()) if ri.size else -1)


@pytest.mark.parametrize("text,line", [("1 2\n3 x\n", 2), ("1 2\n\n3 -4\n", 3), ("1.5\n", 1)])
def test_native_reader_errors_are_the_reference_errors(tmp_path, text, line):
    p = tmp_path / "bad.dat"
    p.write_text(text, encoding="utf-8")
    with pytest.raises(crop.ParseError) as e:
        sparse.read_fimi_csr(p)
    assert e.value.line_no == line
    with pytest.raises(crop.ParseError) as e2:
        sparse.read_fimi(p)
    assert str(e.value) == str(e2.value)


def test_native_reader_large_random_file(tmp_path):
    rng = np.random.default_rng(1)
    p = tmp_path / "big.dat"
    with open(p, "w") as fh:
        for _ in range(200_000):
            n = int(rng.integers(0, 25))
            fh.write(" ".join(str(x) for x in rng.integers(0, 3000, size=n)) + "\n")
    for threads in (1, 3, 0):
        off, items, _ = sparse.read_fimi_csr(p, threads=threads)
        ro, ri = _python_csr(p)
        assert np.array_equal(off, ro) and np.array_equal(items, ri)


def test_fimi_stream_matches_transactions_to_stream(tmp_path):
    p = tmp_path / "m.dat"
    p.write_text("0 1 2\n1 2\n2 3 3\n", encoding="utf-8")
    a = mining.fimi_stream(p)
    b = mining.transactions_to_stream(sparse.read_fimi(p))
    assert a.n_rows == b.n_rows and np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.items, b.items)
    with pytest.raises(crop.InputError):
        mining.fimi_stream(p, dim=3)


# ---------------------------------------------------------------- triple files

def _write(path, text):
    with open(path, "w", newline="") as fh:
        fh.write(text)


def test_native_triple_reader_matches_reference(golden, tmp_path):
    """load_column_row_streams through the native reader (csrc/ingest.cu)
    gives the reference's stream; malformed files raise the reference's
    ParseError (same line number and message) through the fallback."""
    from paper_1210_0461_b200 import sparse

    for n, case in enumerate(golden["triples"]):
        pa, pb = tmp_path / f"a{n}.t", tmp_path / f"b{n}.t"
        _write(pa, case["a"])
        if not case.get("side_only"):
            _write(pb, case["b"])
            s = crop.load_column_row_streams(pa, pb)
            got = [[list(a.indices), list(a.values), list(b.indices), list(b.values)] for a, b in s]
            assert got == case["products"]
            assert s.zero_values_dropped == case["zeros"]
            continue
        if case["ok"]:
            r, c, ptr, idx, val, zeros = sparse.read_triple_csr(pa)
            assert [r, c] == case["header"] and zeros == case["zeros"]
            groups = [[[int(i), float(v)] for i, v in zip(idx[ptr[k]:ptr[k + 1]], val[ptr[k]:ptr[k + 1]])]
                      for k in range(ptr.shape[0] - 1)]
            assert groups == case["groups"]
        else:
            with pytest.raises(crop.ParseError) as exc:
                sparse.read_triple_csr(pa)
            assert exc.value.line_no == case["line_no"]
            assert str(exc.value).split(": ", 1)[1] == case["message"]


def test_native_triple_reader_large_multithreaded(tmp_path):
    """A file big enough to be cut into many thread chunks: the CSR equals
    the reference-exact Python reader's groups."""
    from paper_1210_0461_b200 import sparse

    rng = np.random.default_rng(4)
    n_vec, dim = 30_000, 5_000
    lines = [f"{dim} {dim} {n_vec}"]
    for k in range(n_vec):
        idx = rng.choice(dim, rng.integers(0, 9), replace=False)
        for i in idx:  # unsorted within k, sorted by the reader
            lines.append(f"{k} {int(i)} {float(rng.standard_normal())!r}")
    p = tmp_path / "big.t"
    _write(p, "\n".join(lines) + "\n")
    r, c, ptr, idx, val, zeros = sparse.read_triple_csr(p, threads=8)
    r2, c2, groups, z2 = sparse.read_triple_file(p)
    assert (r, c, zeros) == (r2, c2, z2)
    assert ptr.shape[0] == n_vec + 1
    for k in range(0, n_vec, 997):
        g = groups[k]
        assert idx[ptr[k]:ptr[k + 1]].tolist() == [i for i, _ in g]
        assert val[ptr[k]:ptr[k + 1]].tolist() == [v for _, v in g]
    # an unsorted k far into the file is found through the fallback
    lines.insert(len(lines) // 2, f"0 1 1.0")
    _write(p, "\n".join(lines) + "\n")
    with pytest.raises(crop.ParseError):
        sparse.read_triple_csr(p, threads=8)
