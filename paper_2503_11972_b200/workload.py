"""Vectorised synthetic inputs for parity tests and the benchmark.

Same generative model as the reference's generators (pkg/src/mixserve/
workload.py:93-154): queries are unit vectors scattered around cluster
centres on the sphere (``normalize(center + spread * g)``), cached images
are ``normalize(beta * q + (1 - beta) * g')``, and spread scales as
0.0554 * sqrt(384 / D) so the within-cluster similarity stays in the
0.25-0.30 threshold band at every D (SURVEY.md §8 d).  These streams are NOT
bit-identical to numpy's per-record generator — golden parity uses the
reference's own outputs (tests/golden) — they exist to build 100k-10M entry
caches quickly.
"""
from __future__ import annotations

import math

import numpy as np

# calibrate_beta(0.311) at seed 17 (SURVEY.md §8 d)
CALIBRATED_BETA = {384: 0.947265625, 768: 0.962890625, 1024: 0.966796875}


def spread_for(dim: int) -> float:
    return 0.0554 * math.sqrt(384.0 / dim)


def beta_for(dim: int) -> float:
    return CALIBRATED_BETA.get(dim, 0.96)


def _unit_rows(m: np.ndarray) -> np.ndarray:
    return m / np.linalg.norm(m, axis=1, keepdims=True)


class ClusteredWorkload:
    """Cluster centres + query / image samplers with DiffusionDB-like locality."""

    def __init__(self, dim: int, n_clusters: int = 512, seed: int = 17, spread: float | None = None,
                 beta: float | None = None):
        self.dim = dim
        self.rng = np.random.default_rng(seed)
        self.centers = _unit_rows(self.rng.standard_normal((n_clusters, dim)))
        self.spread = spread_for(dim) if spread is None else spread
        self.beta = beta_for(dim) if beta is None else beta

    def queries(self, n: int, clusters: np.ndarray | None = None) -> np.ndarray:
        idx = self.rng.integers(0, len(self.centers), n) if clusters is None else clusters
        return _unit_rows(self.centers[idx] + self.spread * self.rng.standard_normal((n, self.dim)))

    def images(self, q: np.ndarray) -> np.ndarray:
        return _unit_rows(self.beta * q + (1.0 - self.beta) * self.rng.standard_normal(q.shape))

    def cache_rows(self, n: int, chunk: int = 65536) -> np.ndarray:
        out = np.empty((n, self.dim), dtype=np.float64)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            out[s:e] = self.images(self.queries(e - s))
        return out


def near_threshold_queries(rows: np.ndarray, taus, rng: np.random.Generator, n: int,
                           offsets=(0.0, 1e-9, -1e-9, 1e-6, -1e-6)) -> np.ndarray:
    """q = s e + sqrt(1 - s^2) u with u ⟂ e, s = tau + offset (test_scheduler.py:20-22 generalised)."""
    d = rows.shape[1]
    out = np.empty((n, d))
    for i in range(n):
        e = rows[rng.integers(0, rows.shape[0])]
        u = rng.standard_normal(d)
        u -= (u @ e) * e
        u /= np.linalg.norm(u)
        s = taus[i % len(taus)] + offsets[(i // len(taus)) % len(offsets)]
        out[i] = s * e + math.sqrt(1.0 - s * s) * u
    return out


class GeneratedWorkload:
    """The same generative model with the cache rows generated ON THE DEVICE (mc_generate_rows,
    SURVEY.md §8 f4): 1M-10M entry caches without building them on the host.  Cluster centres
    and queries come from numpy; row r's cluster and noise come from a counter hash on the GPU,
    so the rows are not numpy's streams — parity checks read them back (DeviceRing.read_rows)."""

    def __init__(self, dim: int, n_clusters: int = 512, seed: int = 17, spread: float | None = None,
                 beta: float | None = None):
        self.dim = dim
        self.seed = seed
        self.rng = np.random.default_rng(seed)
        self.centers = _unit_rows(self.rng.standard_normal((n_clusters, dim)))
        self.spread = spread_for(dim) if spread is None else spread
        self.beta = beta_for(dim) if beta is None else beta

    def fill(self, ring, n: int, row0: int = 0) -> None:
        ring.generate(n, self.centers, self.spread, self.beta, self.seed, row0)

    def queries(self, n: int) -> np.ndarray:
        idx = self.rng.integers(0, len(self.centers), n)
        return _unit_rows(self.centers[idx] + self.spread * self.rng.standard_normal((n, self.dim)))

    def trace_queries(self, n: int, active: int = 64, turnover: int = 256) -> np.ndarray:
        """Queries with temporal locality, the reference's cluster lifetimes vectorised
        (workload.py:93-121): request i draws its cluster from a window of `active` clusters that
        advances by one cluster every `turnover` requests, so popular prompts recur for a while
        and then fade."""
        idx = (np.arange(n) // turnover + self.rng.integers(0, active, n)) % len(self.centers)
        return _unit_rows(self.centers[idx] + self.spread * self.rng.standard_normal((n, self.dim)))

    def images(self, q: np.ndarray) -> np.ndarray:
        """Generated-image embeddings for queries q (workload.py:141-154's model)."""
        return _unit_rows(self.beta * q + (1.0 - self.beta) * self.rng.standard_normal(q.shape))
