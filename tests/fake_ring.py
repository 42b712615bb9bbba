"""CPU stand-in for the device ring — TEST INFRASTRUCTURE for host-logic tests only.

It lets the CPU suite exercise SemanticCache's host logic (validation order,
eviction bookkeeping, result mapping) without a GPU.  It mirrors the ring's
FIFO semantics with a numpy float64 window and answers lookups with the
oracle's scan formula.  The product never uses it.
"""
import numpy as np

from oracle.retrieval import OracleTable
from paper_2503_11972_b200 import _native


class FakeRing:
    def __init__(self, capacity, dim, device=0):
        self.capacity, self.dim = capacity, dim
        self.rows = []
        self.pairs = None
        self.appends = 0
        self.evictions = 0

    def close(self):
        pass

    def set_table(self, pairs, total_steps):
        self.pairs = tuple(pairs)
        self.total_steps = int(total_steps)

    def set_sigma_schedule(self, schedule):
        self.schedule = None if schedule is None else np.asarray(schedule, dtype=np.float64)

    def decisions(self, Q):
        """The device epilogue's serving decision, restated (merge.cuh decide): steps = T - k
        (engine.py:38-45), route (scheduler.py:80-89), sigma[k] (cache.py:325-334)."""
        live, sim, k, flags = self.retrieve(Q)
        out = np.zeros(len(live), dtype=_native.DECISION_DTYPE)
        out["live"], out["similarity"], out["k"], out["flags"] = live, sim, k, flags
        hit = (flags & _native.MC_FLAG_HIT) != 0
        out["route"] = hit
        out["steps"] = np.where(hit, self.total_steps - k, self.total_steps)
        sched = getattr(self, "schedule", None)
        out["sigma"] = np.nan
        if sched is not None:
            ok = hit & (k > 0) & (k < len(sched))
            out["sigma"][ok] = sched[k[ok]]
        return out

    def append(self, rows):
        rows = np.asarray(rows, dtype=np.float64).reshape(-1, self.dim)
        for r in rows:
            if len(self.rows) == self.capacity:
                self.rows.pop(0)
            self.rows.append(r.copy())
            self.appends += 1

    def append1(self, row):
        self.append(row)

    def retrieve1(self, q):
        live, sim, k, flags = self.retrieve(np.asarray(q, dtype=np.float64)[None, :])
        return int(live[0]), float(sim[0]), int(k[0]), int(flags[0])

    def submit1(self, q):
        # answered against the rows as they are now; like the native ring, at most three single
        # queries in flight (two beside a batch)
        pend = self.__dict__.setdefault("_inflight", {})
        batches = self.__dict__.setdefault("_batch_tickets", set())
        assert len(pend) < 3 and not (len(pend) >= 2 and batches & set(pend)), "too many lookups in flight"
        self._ticket = getattr(self, "_ticket", 6) + 1
        pend[self._ticket] = self.retrieve1(q)
        return self._ticket

    def wait1(self, ticket):
        return self._inflight.pop(ticket)

    def submit(self, Q):
        pend = self.__dict__.setdefault("_inflight", {})
        assert len(pend) < 2, "a third lookup submitted while two are in flight"
        self._ticket = getattr(self, "_ticket", 6) + 1
        pend[self._ticket] = self.retrieve(Q)
        self.__dict__.setdefault("_batch_tickets", set()).add(self._ticket)
        return self._ticket

    def wait(self, ticket, B):
        out = self._inflight.pop(ticket)
        assert len(out[0]) == B
        return out

    def evict_front(self, n):
        assert 0 <= n <= len(self.rows)
        del self.rows[:n]
        self.evictions += n

    def __len__(self):
        return len(self.rows)

    def retrieve(self, Q):
        Q = np.asarray(Q, dtype=np.float64)
        t = OracleTable(self.pairs)
        m = np.stack(self.rows)
        out = [], [], [], []
        for q in Q:
            sims = m @ q
            best = float(sims.max())
            live = int(np.flatnonzero(sims == best)[-1])
            k = t.select_k(best)
            flags = 0 if best < t.tau else _native.MC_FLAG_HIT
            for lst, v in zip(out, (live, best, k or 0, flags)):
                lst.append(v)
        return tuple(np.array(x) for x in out)
