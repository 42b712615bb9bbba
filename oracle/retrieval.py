"""CPU oracle for the MoDM cache-retrieval hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy float64, the reference's retrieval algorithm so
that the CUDA path can be checked against it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it; the product package never does.

What is restated (reference = /root/reference/pkg/src/mixserve/cache.py):

* ``OracleTable.select_k``     — cache.py:112-117 (largest k with sim >= tau_k)
* ``OracleTable.tau``          — cache.py:103-106 (lowest tau = hit threshold)
* ``OracleCache`` storage      — cache.py:147-168 (state), :181-192
  (``_append_row``: append at _hi, compact when live <= half, else double),
  :194-196 (evict front), :198-235 (policy / validation / age evict /
  capacity evict), :237-242 (``add``)
* ``OracleCache.retrieve``     — cache.py:244-260: float64 ``window @ q``
  (numpy -> OpenBLAS dgemv, the same library call the reference makes),
  newest-among-ties argmax via the reversed view, miss below ``tau`` with
  the similarity still returned.
* ``scan_oracle``              — the reference's *independent* scan formula
  from pkg/tests/test_acceptance.py:429-436 (own matrix, max, last argmax,
  k = max k with sim >= tau) used where the per-row store is too slow.

Pinning: ``tests/golden/make_golden.py`` runs the real reference (importable
from /root/reference in the build container) over seeded op logs and stores
its outputs in ``tests/golden/*.npz``; ``tests/test_oracle.py`` replays the
logs through this oracle and requires identical decisions and similarities
bit-identical to the reference's own floats.

Dependency note: the arithmetic lives in numpy -> OpenBLAS ``dgemv``
(third-party, pinned only as ``numpy>=1.24`` in pkg/pyproject.toml:9).  This
image has numpy 2.3.5 with scipy-openblas 0.3.30; ``blas_info()`` reports it.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np

NORM_TOL = 1e-6  # cache.py:28
PRODUCERS = ("large", "small")  # cache.py:20-21
POLICIES = ("all", "large", "disabled")  # cache.py:23-26
DEFAULT_PAIRS = ((5, 0.25), (10, 0.26), (15, 0.27), (20, 0.28), (25, 0.29), (30, 0.30))  # cache.py:18


class OracleTable:
    """(k, tau_k) pairs; restates ThresholdTable (cache.py:73-117) minus validation."""

    def __init__(self, pairs=DEFAULT_PAIRS, total_steps: int = 50):
        self.pairs = tuple((int(k), float(t)) for k, t in pairs)
        self.total_steps = int(total_steps)

    @property
    def tau(self) -> float:  # cache.py:103-106
        return self.pairs[0][1]

    def select_k(self, sim: float):  # cache.py:112-117
        best = None
        for k, t in self.pairs:  # ascending; last satisfied wins == reversed first
            if sim >= t:
                best = k
        return best


@dataclass(frozen=True)
class OracleEntry:
    id: str
    embedding: np.ndarray
    producer: str
    seq: int
    inserted_at: float


class OracleCache:
    """FIFO store + exhaustive float64 scan, restating SemanticCache.

    The growable window (``_rows``/``_lo``/``_hi``) follows cache.py:165,
    181-196 exactly, because OpenBLAS's summation order — and therefore the
    last ulp of each similarity — depends on where the live window sits in
    its buffer (SURVEY.md §0 finding 3).
    """

    def __init__(self, capacity: int, dim: int, policy: str = "all", max_age_s=None):
        if capacity < 1 or policy not in POLICIES:
            raise ValueError("bad oracle cache config")
        self.capacity = int(capacity)
        self.dim = int(dim)
        self.policy = policy
        self.max_age_s = max_age_s
        self.meta: deque[OracleEntry] = deque()
        self._rows = np.empty((min(self.capacity, 1024), self.dim), dtype=np.float64)
        self._lo = 0
        self._hi = 0
        self.next_seq = 0

    def __len__(self):
        return len(self.meta)

    # -- storage (cache.py:181-196) -----------------------------------------
    def _push_row(self, emb: np.ndarray) -> None:
        cap_rows = self._rows.shape[0]
        if self._hi == cap_rows:
            live = self._hi - self._lo
            if live <= cap_rows // 2:
                self._rows[:live] = self._rows[self._lo:self._hi]
            else:
                bigger = np.empty((max(1024, cap_rows * 2), self.dim), dtype=np.float64)
                bigger[:live] = self._rows[self._lo:self._hi]
                self._rows = bigger
            self._lo, self._hi = 0, live
        self._rows[self._hi] = emb
        self._hi += 1

    def _pop_front(self) -> OracleEntry:
        self._lo += 1
        return self.meta.popleft()

    # -- mutation (cache.py:198-242) ----------------------------------------
    def admits(self, producer: str) -> bool:
        return self.policy == "all" or (self.policy == "large" and producer == "large")

    def insert(self, e: OracleEntry) -> list:
        if not self.admits(e.producer):
            return []
        if e.producer not in PRODUCERS:
            raise ValueError("producer")
        if e.embedding.shape != (self.dim,):
            raise ValueError("shape")
        if abs(float(np.linalg.norm(e.embedding)) - 1.0) > NORM_TOL:
            raise ValueError("norm")
        if self.meta and e.seq <= self.meta[-1].seq:
            raise ValueError("seq")
        out = []
        if self.max_age_s is not None:
            horizon = e.inserted_at - self.max_age_s
            while self.meta and self.meta[0].inserted_at < horizon:
                out.append(self._pop_front())
        self.meta.append(e)
        self._push_row(e.embedding)
        while len(self.meta) > self.capacity:
            out.append(self._pop_front())
        self.next_seq = max(self.next_seq, e.seq + 1)
        return out

    def add(self, id, embedding, producer, inserted_at):
        return self.insert(OracleEntry(id, embedding, producer, self.next_seq, inserted_at))

    # -- the hot path (cache.py:244-260) ------------------------------------
    def scores(self, q: np.ndarray) -> np.ndarray:
        return self._rows[self._lo:self._hi] @ q

    def retrieve(self, q: np.ndarray, table: OracleTable):
        """Returns (live_index | None, similarity | None, k | None)."""
        if q.shape != (self.dim,):
            raise ValueError("query shape")
        if not self.meta:
            return None, None, None
        sims = self.scores(q)
        n = sims.shape[0]
        live = n - 1 - int(np.argmax(sims[::-1]))  # newest among equal maxima
        best = float(sims[live])
        if best < table.tau:
            return None, best, None
        return live, best, table.select_k(best)

    def retrieve_entry(self, q, table):
        live, sim, k = self.retrieve(q, table)
        return (self.meta[live] if live is not None else None), sim, k


def scan_oracle(matrix: np.ndarray, q: np.ndarray, table: OracleTable):
    """Independent scan formula of test_acceptance.py:429-436.

    Returns (live_index | None, similarity, k | None, best_live_index).
    """
    sims = matrix @ q
    best = float(sims.max())
    idx = int(np.flatnonzero(sims == best)[-1])
    if best < table.tau:
        return None, best, None, idx
    return idx, best, max(k for k, t in table.pairs if best >= t), idx


def ambiguity(matrix: np.ndarray, q: np.ndarray, table: OracleTable, band: float = 1e-12):
    """Flags the cases the north star says must be *reported*, not asserted.

    tie:        two or more rows share the maximal float64 score exactly
    near_tie:   runner-up within ``band`` of the best (but not equal)
    near_tau:   best within ``band`` of any tau_k
    """
    sims = matrix @ q
    order = np.argsort(sims)
    best = sims[order[-1]]
    second = sims[order[-2]] if sims.shape[0] > 1 else -np.inf
    return {
        "tie": bool(second == best),
        "near_tie": bool(second != best and best - second < band),
        "near_tau": bool(any(abs(best - t) < band for _, t in table.pairs)),
    }


def blas_info() -> str:
    try:
        cfg = np.show_config(mode="dicts")
        blas = cfg["Build Dependencies"]["blas"]
        return f"numpy {np.__version__}, {blas.get('name')} {blas.get('version')}"
    except Exception:  # pragma: no cover - informational only
        return f"numpy {np.__version__}"
