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
