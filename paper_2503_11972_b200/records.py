"""Value types and small helpers of the cache API (the non-device part).

These are the symbols the reference exports next to ``SemanticCache``
(pkg/src/mixserve/__init__.py:15-24; definitions in pkg/src/mixserve/cache.py).
Their observable behaviour — field layout, validation order, exception types
and message texts — is part of the drop-in contract, so callers and the
reference's own tests cannot tell the two apart.  Citations give the
reference line each rule mirrors.
"""
from __future__ import annotations

from collections.abc import Sequence as _SequenceABC
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

DEFAULT_DIM = 512                                  # cache.py:16
STEP_CHOICES = (5, 10, 15, 20, 25, 30)              # cache.py:17
DEFAULT_THRESHOLDS = tuple(zip(STEP_CHOICES, (0.25, 0.26, 0.27, 0.28, 0.29, 0.30)))  # cache.py:18

LARGE, SMALL = "large", "small"                     # cache.py:20-21
POLICY_ALL, POLICY_LARGE, POLICY_DISABLED = "all", "large", "disabled"  # cache.py:23-25
POLICIES = (POLICY_ALL, POLICY_LARGE, POLICY_DISABLED)                  # cache.py:26
NORM_TOL = 1e-6                                     # cache.py:28


class EmbeddingError(ValueError):
    """Raised for vectors that cannot serve as embeddings."""


def normalize(v: Sequence[float] | np.ndarray) -> np.ndarray:
    """Unit-length float64 copy of a finite, nonzero 1-d vector (cache.py:35-48)."""
    vec = np.asarray(v, dtype=np.float64)
    if vec.ndim != 1:
        raise EmbeddingError(f"expected 1-d vector, got shape {vec.shape}")
    if not np.isfinite(vec).all():
        raise EmbeddingError("vector has non-finite components")
    length = float(np.linalg.norm(vec))
    if length == 0.0:
        raise EmbeddingError("cannot normalize the zero vector")
    return vec / length


def cosine(q: np.ndarray, e: np.ndarray) -> float:
    """Similarity of two unit embeddings = their dot product (cache.py:51-55)."""
    if q.shape != e.shape:
        raise EmbeddingError(f"dimension mismatch: {q.shape} vs {e.shape}")
    return float(np.dot(q, e))


def is_normalized(v: np.ndarray, tol: float = NORM_TOL) -> bool:
    """|‖v‖₂ − 1| ≤ tol (cache.py:58-59)."""
    return abs(float(np.linalg.norm(v)) - 1.0) <= tol


@dataclass(frozen=True)
class CacheEntry:
    """One cached generation: embedding plus provenance (cache.py:62-70)."""

    id: str
    embedding: np.ndarray
    producer: str  # LARGE or SMALL
    seq: int
    inserted_at: float  # simulated seconds


@dataclass(frozen=True)
class RetrievalResult:
    """What a lookup returns (cache.py:120-130): a hit carries the entry and k;
    a miss carries only the best similarity (or nothing, for an empty cache)."""

    entry: CacheEntry | None
    similarity: float | None
    k: int | None

    @property
    def hit(self) -> bool:
        return self.entry is not None


def _result_factory(cls=None):
    """A constructor for RetrievalResult (or another frozen dataclass with the same three
    fields, e.g. the host application's own) that skips the frozen dataclass's per-field
    object.__setattr__ calls (about half the cost of a batch's result objects).  The
    instances are ordinary `cls` objects: same fields, equality, hash and repr."""
    new = object.__new__
    cls = RetrievalResult if cls is None else cls

    def make(entry, similarity, k):
        r = new(cls)
        d = r.__dict__
        d["entry"] = entry
        d["similarity"] = similarity
        d["k"] = k
        return r

    return make


make_result = _result_factory()


def _entry_factory(cls=None):
    """A constructor for CacheEntry (or the host application's frozen dataclass with the same
    five fields) that fills the instance dict directly instead of five object.__setattr__
    calls; add() mints one entry per request.  The objects are ordinary `cls` instances."""
    new = object.__new__
    cls = CacheEntry if cls is None else cls

    def make(id, embedding, producer, seq, inserted_at):
        e = new(cls)
        d = e.__dict__
        d["id"] = id
        d["embedding"] = embedding
        d["producer"] = producer
        d["seq"] = seq
        d["inserted_at"] = inserted_at
        return e

    return make


make_entry = _entry_factory()


class RetrievalBatch(_SequenceABC):
    """The answers of one batched lookup (SemanticCache.retrieve_batch): a read-only sequence
    of RetrievalResult, equal to the list B retrieve() calls return, whose objects are built on
    first access (the hit entries are captured at lookup time, so later inserts and evictions
    do not change them), plus the answers as arrays: ``similarity`` (float64, NaN on an empty
    cache), ``k`` (int32, 0 = none) and ``hit`` (bool)."""

    __slots__ = ("_ents", "similarity", "k", "flags", "_items", "_make", "_miss")

    def __init__(self, ents, similarity, k, flags, make, miss):
        self._ents = ents
        self.similarity = similarity
        self.k = k
        self.flags = flags
        self._items = None
        self._make = make
        self._miss = miss

    @property
    def hit(self):
        return (self.flags & 1) != 0

    def __len__(self) -> int:
        return len(self._ents)

    def _build(self):
        make, miss = self._make, self._miss
        out = []
        for e, s, kk, f in zip(self._ents, self.similarity.tolist(), self.k.tolist(), self.flags.tolist()):
            if e is not None:
                out.append(make(e, s, kk or None))
            elif f & 2:  # empty cache
                out.append(miss)
            else:
                out.append(make(None, s, None))
        self._items = out
        return out

    def __getitem__(self, i):
        items = self._items if self._items is not None else self._build()
        return items[i]

    def __iter__(self):
        items = self._items if self._items is not None else self._build()
        return iter(items)

    def __eq__(self, other):
        if isinstance(other, RetrievalBatch):
            other = list(other)
        if not isinstance(other, (list, tuple)):
            return NotImplemented
        return list(self) == list(other)

    def __repr__(self) -> str:
        return f"RetrievalBatch({list(self)!r})"


class ThresholdTable:
    """Similarity thresholds tau_k per skippable step count k (cache.py:73-117).

    The first (lowest) tau is the hit threshold; ``select_k`` returns the
    largest k whose tau the similarity reaches.  The device epilogue applies
    the same rule to the float64 similarity it certifies.
    """

    def __init__(self, pairs: Iterable[tuple[int, float]], total_steps: int = 50):
        table = [(int(k), float(tau)) for k, tau in pairs]
        if not table:
            raise ValueError("threshold table must not be empty")
        ks = [k for k, _ in table]
        taus = [tau for _, tau in table]
        # the reference's predicates, evaluated lazily in its order (cache.py:84-93): a NaN
        # tau passes `b <= a` and is caught by the range check, as there
        if _falls(ks):
            raise ValueError(f"k values must be strictly increasing: {ks}")
        if _falls(taus):
            raise ValueError(f"thresholds must be strictly increasing: {taus}")
        if any(not -1.0 <= t <= 1.0 for t in taus):
            raise ValueError(f"thresholds must lie in [-1, 1]: {taus}")
        if ks[-1] >= total_steps:
            raise ValueError(f"max k {ks[-1]} must stay below total steps {total_steps}")
        if any(k <= 0 for k in ks):
            raise ValueError(f"k values must be positive: {ks}")
        self.pairs = tuple(table)
        self.total_steps = int(total_steps)

    @classmethod
    def default(cls, total_steps: int = 50) -> "ThresholdTable":
        return cls(DEFAULT_THRESHOLDS, total_steps=total_steps)

    @property
    def tau(self) -> float:
        """Global hit threshold: the lowest per-k threshold."""
        return self.pairs[0][1]

    @property
    def step_choices(self) -> tuple[int, ...]:
        return tuple(k for k, _ in self.pairs)

    def select_k(self, similarity: float) -> int | None:
        """Largest k whose threshold the similarity meets, or None."""
        met = [k for k, tau in self.pairs if similarity >= tau]
        return met[-1] if met else None


def _falls(values: list) -> bool:
    """Some neighbour fails to rise (the reference's `any(b <= a ...)`, NaN-tolerant like it)."""
    return any(b <= a for a, b in zip(values, values[1:]))


# -- noise re-entry schedule (cache.py:305-334); exported, not on the lookup path ---------
def linear_sigma_schedule(total_steps: int) -> np.ndarray:
    """sigma(t) = 1 - t/T for t = 0..T."""
    if total_steps < 1:
        raise ValueError(f"total_steps must be >= 1, got {total_steps}")
    return 1.0 - np.arange(total_steps + 1, dtype=np.float64) / total_steps


def validate_sigma_schedule(schedule: np.ndarray) -> None:
    """Endpoints 1 -> 0, non-increasing, values within [0, 1]."""
    sig = np.asarray(schedule, dtype=np.float64)
    if sig.ndim != 1 or sig.shape[0] < 2:
        raise ValueError("schedule must be a 1-d table over timesteps 0..T")
    if sig[0] != 1.0 or sig[-1] != 0.0:
        raise ValueError("schedule must start at 1.0 and end at 0.0")
    if (np.diff(sig) > 0).any():
        raise ValueError("schedule must be non-increasing")
    if (sig < 0.0).any() or (sig > 1.0).any():
        raise ValueError("schedule values must lie in [0, 1]")


def noise_reentry_level(k: int, schedule: np.ndarray) -> float:
    """Noise level at which refinement of a cached image resumes after skipping k steps."""
    last = len(schedule) - 1
    if not 0 <= k <= last:
        raise ValueError(f"k={k} outside the schedule range [0, {last}]")
    return float(schedule[k])
