import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")) as fh:
        return json.load(fh)


def tx_to_csr(transactions):
    import numpy as np
    lens = np.array([len(t) for t in transactions], dtype=np.int64)
    offsets = np.zeros(len(transactions) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    items = np.array([i for t in transactions for i in t], dtype=np.uint32)
    return offsets, items


def vectors_to_csr(vecs):
    import numpy as np
    lens = np.array([len(ix) for ix, _ in vecs], dtype=np.int64)
    ptr = np.zeros(len(vecs) + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    idx = np.array([i for ix, _ in vecs for i in ix], dtype=np.uint32)
    val = np.array([v for _, vs in vecs for v in vs], dtype=np.float64)
    return ptr, idx, val
