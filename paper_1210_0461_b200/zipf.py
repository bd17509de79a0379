"""Synthetic Zipf workloads under the reference's names (oracle.py:74-185).

`ZipfModel`, `gen_zipf_stream` and `gen_zipf_transactions` are part of the
reference's public API (`__init__.py:60-65`) even though they only build
inputs. They are restated here draw for draw: the same `random.Random` /
`numpy.random.default_rng` calls in the same order, so a seed gives the same
stream or transaction list as the reference (pinned by
tests/test_host.py against reference-generated fixtures). They are host-side
input builders, not part of the measured path; the bench's BASELINE-shaped
workloads come from `workloads.py`.
"""

import random
from dataclasses import dataclass

from .errors import ConfigError
from .sparse import OuterProductStream, SparseVector, write_fimi


@dataclass(frozen=True)
class ZipfModel:
    """Ranked weights: rank r (1-based) weighs scale / r**skew (oracle.py:74-94)."""

    scale: float
    skew: float
    distinct: int

    def __post_init__(self):
        for name, ok in (("scale", self.scale > 0), ("skew", self.skew > 0)):
            if not ok:
                raise ConfigError(f"{name} must be positive, got {getattr(self, name)}")
        if self.distinct < 1:
            raise ConfigError(f"distinct must be >= 1, got {self.distinct}")

    def rank_weight(self, rank: int) -> float:
        return self.scale / rank ** self.skew

    def weights(self) -> list[float]:
        return [self.rank_weight(r) for r in range(1, self.distinct + 1)]


def gen_zipf_stream(model: ZipfModel, dim: int, outer_count: int | None,
                    seed: int) -> OuterProductStream:
    """A stream whose exact product carries the model's weights on `distinct`
    random cells of [0, dim)^2 (oracle.py:97-150).

    Every product is (unit row vector) x (that row's weights / copies), so no
    product touches a cell outside the chosen set. outer_count == distinct
    gives one rank-1 product per cell; None one product per occupied row;
    otherwise the extra products go round-robin over the sorted rows."""
    d = model.distinct
    if d > dim * dim:
        raise ConfigError(f"cannot place {d} distinct entries in a {dim}x{dim} product")
    cells = random.Random(seed).sample(range(dim * dim), d)
    weights = model.weights()
    if outer_count == d:
        return OuterProductStream.from_pairs(dim, dim, [
            (SparseVector(dim, [c // dim], [1.0]), SparseVector(dim, [c % dim], [w]))
            for c, w in zip(cells, weights)])
    per_row: dict[int, list] = {}
    for c, w in zip(cells, weights):
        per_row.setdefault(c // dim, []).append((c % dim, w))
    rows = sorted(per_row)
    n_out = len(rows) if outer_count is None else outer_count
    if n_out < len(rows):
        raise ConfigError(f"outer_count={outer_count} infeasible: need at least one product "
                          f"per occupied row ({len(rows)})")
    base, extra = divmod(n_out - len(rows), len(rows)) if rows else (0, 0)
    products = []
    for k, row in enumerate(rows):
        copies = 1 + base + (1 if k < extra else 0)
        cols = sorted(per_row[row])
        left = SparseVector(dim, [row], [1.0])
        right = SparseVector(dim, [j for j, _ in cols], [w / copies for _, w in cols])
        products += [(left, right)] * copies
    return OuterProductStream.from_pairs(dim, dim, products)


def gen_zipf_transactions(item_count: int, tx_count: int, skew: float, seed: int,
                          mean_size: int = 10, path=None) -> list[tuple[int, ...]]:
    """Transactions with Zipf item popularity (oracle.py:153-185): per
    transaction 2 + Poisson(mean_size - 2) draws with replacement from
    p(r) ~ 1/r**skew, de-duplicated and sorted. Writes a FIMI file when
    `path` is given."""
    if item_count < 1 or tx_count < 0 or mean_size < 1:
        raise ConfigError("item_count >= 1, tx_count >= 0, mean_size >= 1 required")
    if skew <= 0:
        raise ConfigError(f"skew must be positive, got {skew}")
    import numpy as np

    gen = np.random.default_rng(seed)
    p = 1.0 / np.arange(1, item_count + 1, dtype=float) ** skew
    p /= p.sum()
    lam = max(mean_size - 2, 0)
    out = []
    for _ in range(tx_count):
        size = min(2 + gen.poisson(lam), item_count)
        drawn = gen.choice(item_count, size=size, p=p)
        out.append(tuple(int(x) for x in np.unique(drawn)))
    if path is not None:
        write_fimi(path, out)
    return out
