"""CPU stand-in for one shard's device ring — TEST INFRASTRUCTURE for the gloo tests.

Mirrors the native ring's shard contract: local rows are the
shard's global positions p ≡ g (mod G) in FIFO order; ``retrieve_local_async``
writes one 32-byte mc_record per query (float64 best, runner-up, global
position, flags) into a CPU uint8 tensor, and ``merge_records`` restates
k_finalize (csrc/rescore.cu): max similarity, ties to the larger position,
then the threshold / k rule of cache.py:255-260 and :112-117.  Scores come
from the oracle's numpy float64 scan, so the merged answer must equal the
single-cache oracle's.
"""
import numpy as np
import torch

from oracle.retrieval import OracleTable
from paper_2503_11972_b200 import _native

REC = np.dtype([("sim", "<f8"), ("second", "<f8"), ("pos", "<i8"), ("flags", "<u4"), ("reserved", "<i4")])


class FakeShardRing:
    def __init__(self, capacity, dim, device=0):
        self.capacity, self.dim = capacity, dim
        self.rows, self.pos = [], []
        self.G, self.g = 1, 0
        self.j = 0  # local append index
        self.pairs, self.total_steps = None, 50

    def configure_shard(self, G, g):
        self.G, self.g = G, g

    def set_table(self, pairs, total_steps):
        self.pairs, self.total_steps = tuple(pairs), total_steps

    def append1(self, row):
        assert len(self.rows) < self.capacity, "shard ring overflow: evictions must come first"
        self.rows.append(np.asarray(row, dtype=np.float64).copy())
        self.pos.append(self.j * self.G + self.g)
        self.j += 1

    def append(self, rows):
        for r in np.asarray(rows, dtype=np.float64).reshape(-1, self.dim):
            self.append1(r)

    def evict_front(self, n):
        assert 0 <= n <= len(self.rows)
        del self.rows[:n], self.pos[:n]

    def __len__(self):
        return len(self.rows)

    def records_device(self):
        return torch.device("cpu")

    def retrieve_local_async(self, Q, out, stream=0):
        rec = np.zeros(Q.shape[0], dtype=REC)
        rec["pos"] = -1
        rec["sim"] = np.nan
        rec["flags"] = 0xFFFFFFFF
        if self.rows:
            sims = np.stack(self.rows) @ np.asarray(Q, dtype=np.float64).T  # [n, B]
            for b in range(Q.shape[0]):
                s = sims[:, b]
                best = s.max()
                idx = np.flatnonzero(s == best)
                rest = s[s != best]
                rec[b] = (best, rest.max() if rest.size else -np.inf, self.pos[idx[-1]],
                          _native.MC_FLAG_TIE if idx.size > 1 else 0, 0)
        out.copy_(torch.from_numpy(rec.view(np.uint8).copy()))

    NEED = 0x10000  # FLAG_NEED_FALLBACK (mc_internal.cuh): the record asks for the exhaustive rescan

    def retrieve_local_submit(self, Q, out, stream=0):
        """Like the native submit: no rescan behind the scan.  Every third query's record (by a
        per-ring counter) comes back degraded and flagged, as a failed certificate would."""
        self.retrieve_local_async(Q, out, stream)
        rec = out.numpy().view(REC)
        # like the native ring: the window this lookup scanned, for a later rescan of its records
        self.__dict__.setdefault("_windows", {})[out.data_ptr()] = (list(self.rows), list(self.pos))
        self._submits = getattr(self, "_submits", 0) + 1
        for b in range(Q.shape[0]):
            if rec[b]["pos"] >= 0 and (b + self._submits) % 3 == 0:
                rec[b]["sim"] -= 0.5
                rec[b]["flags"] |= self.NEED

    def rescan_local(self, Q, out, stream=0):
        rec = out.numpy().view(REC)
        need = [b for b in range(Q.shape[0]) if rec[b]["pos"] >= 0 and rec[b]["flags"] & self.NEED]
        exact = torch.empty_like(out)
        rows, pos = self.rows, self.pos
        self.rows, self.pos = (list(x) for x in self._windows[out.data_ptr()])  # the scanned window
        try:
            self.retrieve_local_async(Q, exact, stream)
        finally:
            self.rows, self.pos = rows, pos
        ex = exact.numpy().view(REC)
        for b in need:
            rec[b] = ex[b]
            rec[b]["flags"] |= _native.MC_FLAG_FALLBACK
        self.rescans = getattr(self, "rescans", 0) + len(need)

    def merge_records(self, gathered, G, B, p0, stream=0):
        recs = gathered.numpy().view(REC).reshape(G, B)
        t = OracleTable(self.pairs, self.total_steps)
        live = np.full(B, -1, np.int64)
        sim = np.full(B, np.nan)
        k = np.zeros(B, np.int32)
        flags = np.zeros(B, np.uint32)
        for b in range(B):
            cand = [(r["sim"], r["pos"]) for r in recs[:, b] if r["pos"] >= 0]
            if not cand:
                flags[b] = _native.MC_FLAG_EMPTY
                continue
            s, p = max(cand)  # larger similarity, then larger (newer) position
            live[b], sim[b] = p - p0, s
            k[b] = t.select_k(s) or 0
            flags[b] = 0 if s < t.tau else _native.MC_FLAG_HIT
            if any(r["flags"] & self.NEED for r in recs[:, b] if r["pos"] >= 0):
                flags[b] |= _native.MC_FLAG_NEED_RESCAN
        return live, sim, k, flags

    def merge_submit(self, gathered, G, B, p0, stream, slot):
        slots = self.__dict__.setdefault("_slots", {})
        assert slot not in slots, "merge slot still holds an unread result"
        slots[slot] = self.merge_records(gathered, G, B, p0, stream)

    def merge_wait(self, slot):
        return self._slots.pop(slot)

    def close(self):
        pass
