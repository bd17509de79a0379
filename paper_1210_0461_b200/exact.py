"""Exact entry weights on the GPU, under the reference's oracle.py names.

`exact_pair_supports` (oracle.py:61-71), `exact_product` (:20-50) and
`exact_top` (:53-58) are the reference's brute-force ground truth. In this
package they are served by the same device kernels as the engine with a
single bucket (kappa = 1 owns everything), so they scale to the benchmark
sizes; the independent CPU checker lives in oracle/ (tests only).
"""

from collections import Counter

import numpy as np

from .errors import ConfigError, ResourceCapError
from .sparse import ColumnRowStream, OuterProductStream, TransactionStream

DEFAULT_WORK_CAP = 10 ** 12  # the reference's 1e8 desk-scale cap, lifted for the GPU


def exact_pair_supports(transactions, work_cap: int = DEFAULT_WORK_CAP) -> Counter:
    """Support of every unordered item pair (GPU exact count, kappa = 1)."""
    from . import kernels

    ts = transactions if isinstance(transactions, TransactionStream) else \
        TransactionStream.from_transactions([sorted(set(t)) for t in transactions])
    if ts.pair_terms(True) > work_cap:
        raise ResourceCapError(f"pair counting needs more than {work_cap} operations")
    n_items = int(ts.items.max()) + 1 if ts.items.size else 1
    dtx = kernels.DeviceTransactions.from_host(ts.offsets, ts.items, n_items)
    row, col, w = kernels.count_pairs(dtx, True).to_numpy()
    return Counter({(int(r), int(c)): int(x) for r, c, x in zip(row, col, w)})


def exact_product(stream: OuterProductStream, upper_only: bool = False,
                  work_cap: int = DEFAULT_WORK_CAP) -> dict:
    """Entry weights of the streamed product, fp64 in stream order; zeros dropped."""
    from . import kernels

    cr = ColumnRowStream.from_stream(stream)
    if cr.total_pair_count() > work_cap:
        raise ResourceCapError(f"exact product needs more than {work_cap} operations; "
                               "raise work_cap only if you mean it")
    ent = kernels.outer_product(kernels.DeviceOuterStream.from_host(cr), upper_only)
    row, col, w = ent.to_numpy()
    keep = w != 0.0
    return {(int(r), int(c)): float(x) for r, c, x in zip(row[keep], col[keep], w[keep])}


def exact_top(weights: dict, k: int) -> list:
    """True top-k entries by weight; ties by (row, col) ascending."""
    if k < 0:
        raise ConfigError(f"k must be >= 0, got {k}")
    return sorted(weights.items(), key=lambda kv: (-kv[1], kv[0]))[:k]
