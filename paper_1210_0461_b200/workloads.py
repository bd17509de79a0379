"""Seeded synthetic workloads with the shapes of BASELINE.json's five configs.

The reference measures nothing on public data for this path and its paper's
datasets are not available here; these generators stand in with the sizes
and distributions SURVEY.md §8(d) fixes (data seed = config number, engine
seed 0). Transactions are generated ON THE GPU (csrc/gen.cu): successive
sampling without replacement from an integer alias table for the Zipf law
P(id = r) ~ 1/(r+1)^s, lengths from an integer CDF -- every draw a pure
function of (seed, transaction, draw index). Configuration 4 (real-valued
A*B) is generated with numpy on the host.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError


@dataclass(frozen=True)
class PairConfig:
    name: str
    n_tx: int
    n_items: int
    zipf_s: float
    length: tuple  # ("poisson", mean, lo, hi) or ("uniform", lo, hi)
    kappa: int
    workers: int
    ss_capacity: int | None  # None = exact regime
    top_k: int
    seed: int
    gpus: int = 1


@dataclass(frozen=True)
class ProductConfig:
    name: str
    n: int
    lomax_alpha: float
    nnz_scale: float
    nnz_lo: int
    nnz_hi: int
    kappa: int
    seed: int
    gpus: tuple = field(default=(1, 2, 4, 8))


CONFIGS = {
    "c1": PairConfig("c1-exact-pairs-cpu-oracle", 20_000, 2_000, 1.2, ("poisson", 8, 2, 50),
                     4, 4, None, 1000, 1),
    "c2": PairConfig("c2-exact-pairs-1gpu", 2_000_000, 50_000, 1.1, ("poisson", 20, 2, 200),
                     8, 8, None, 1000, 2),
    "c3": PairConfig("c3-heavy-hitter-pairs-8gpu", 50_000_000, 1_000_000, 1.0,
                     ("poisson", 30, 2, 500), 1184, 1184, 65536, 10_000, 3, gpus=8),
    "c4": ProductConfig("c4-real-product", 500_000, 2.0, 4.0, 4, 2000, 1184, 4),
    "c5": PairConfig("c5-skew-pairs-8gpu", 5_000_000, 10_000, 1.5, ("uniform", 50, 300),
                     1184, 1184, None, 1000, 5, gpus=8),
}


def zipf_alias(n_items: int, s: float) -> tuple[np.ndarray, np.ndarray]:
    """Integer alias table (thresholds, aliases) for P(r) ~ (r+1)^-s (Vose)."""
    p = 1.0 / np.arange(1, n_items + 1, dtype=np.float64) ** s
    p /= p.sum()
    scaled = p * n_items
    thresh = np.zeros(n_items, dtype=np.float64)
    alias = np.arange(n_items, dtype=np.int64)
    small = [i for i in range(n_items) if scaled[i] < 1.0]
    large = [i for i in range(n_items) if scaled[i] >= 1.0]
    sc = scaled.tolist()
    while small and large:
        a = small.pop()
        b = large.pop()
        thresh[a] = sc[a]
        alias[a] = b
        sc[b] = sc[b] + sc[a] - 1.0
        (small if sc[b] < 1.0 else large).append(b)
    for i in large + small:
        thresh[i] = 1.0
    t32 = np.minimum(np.floor(thresh * 4294967296.0), 4294967295.0).astype(np.uint32)
    return t32, alias.astype(np.uint32)


def length_cdf(spec: tuple) -> tuple[np.ndarray, int]:
    """Integer CDF over [lo, hi] of the configured transaction length law."""
    if spec[0] == "poisson":
        _, mean, lo, hi = spec
        k = np.arange(0, hi + 1)
        logp = -mean + k * np.log(mean) - np.array([np.sum(np.log(np.arange(1, x + 1))) for x in k])
        pmf = np.exp(logp)
        probs = np.zeros(hi - lo + 1)
        probs[0] = pmf[: lo + 1].sum()
        probs[1:-1] = pmf[lo + 1: hi]
        probs[-1] = max(0.0, 1.0 - probs[:-1].sum())
    elif spec[0] == "uniform":
        _, lo, hi = spec
        probs = np.full(hi - lo + 1, 1.0 / (hi - lo + 1))
    else:
        raise ConfigError(f"unknown length law {spec[0]!r}")
    cdf = np.cumsum(probs)
    c32 = np.minimum(np.round(cdf * 4294967296.0), 4294967295.0).astype(np.uint32)
    c32[-1] = 0xFFFFFFFF
    return c32, lo


def generate_pairs_workload(cfg: PairConfig, n_tx: int | None = None):
    """DeviceTransactions for a pair-mining config (optionally a prefix)."""
    from .kernels import generate_transactions

    n = cfg.n_tx if n_tx is None else int(n_tx)
    alias = zipf_alias(cfg.n_items, cfg.zipf_s)
    cdf, lo = length_cdf(cfg.length)
    return generate_transactions(n, cfg.n_items, alias, cdf, lo, cfg.seed)


def generate_product_workload(cfg: ProductConfig, n_products: int | None = None):
    """Host ColumnRowStream for configuration 4 (A as CSC, B as CSR).

    nnz per column of A / row of B = floor(scale * (Lomax(alpha) + 1)) clipped
    to [lo, hi]; positions uniform without replacement; values N(0,1) rounded
    to fp32 (then carried as float64, exactly)."""
    from .sparse import ColumnRowStream

    rng = np.random.default_rng(cfg.seed)
    k = cfg.n if n_products is None else int(n_products)

    def side():
        nnz = np.floor(cfg.nnz_scale * (rng.pareto(cfg.lomax_alpha, size=k) + 1.0))
        nnz = np.clip(nnz, cfg.nnz_lo, cfg.nnz_hi).astype(np.int64)
        ptr = np.zeros(k + 1, dtype=np.int64)
        np.cumsum(nnz, out=ptr[1:])
        owner = np.repeat(np.arange(k), nnz)
        idx = rng.integers(0, cfg.n, size=int(ptr[-1]))
        while True:  # redraw duplicates inside a vector until none remain
            order = np.lexsort((idx, owner))
            idx, owner = idx[order], owner[order]
            dup = np.zeros(idx.shape[0], dtype=bool)
            dup[1:] = (idx[1:] == idx[:-1]) & (owner[1:] == owner[:-1])
            if not dup.any():
                break
            idx[dup] = rng.integers(0, cfg.n, size=int(dup.sum()))
        vals = rng.standard_normal(idx.shape[0]).astype(np.float32).astype(np.float64)
        vals[vals == 0.0] = 1.0
        return ptr, idx.astype(np.uint32), vals

    ap, ai, av = side()
    bp, bi, bv = side()
    return ColumnRowStream(cfg.n, cfg.n, ap, ai, av, bp, bi, bv)
