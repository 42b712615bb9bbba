"""Entry-sharded cache across GPUs: one process per GPU, records merged over NCCL.

Layout.  Global append position p (0, 1, 2, ... over the
cache's lifetime) decides the owner: shard g of G stores p ≡ g (mod G), as
local row j = p // G of its device ring (``mc_configure_shard``).  Every rank
keeps the full metadata FIFO (the reference's ``_store``, cache.py:164), so
validation, eviction decisions and the returned ``CacheEntry`` objects are
identical on all ranks; only the embeddings are divided.

Two deployments share this code:

* ``group`` mode (default): one process per GPU, the shard = the rank of a
  torch.distributed group.  A lookup is SPMD: every rank passes the same
  query batch, scans its shard with the certified local scan (``mc_retrieve_local_async`` -> one 32-byte
``mc_record`` per query: exact float64 best, runner-up, global position,
flags), the records are all-gathered (``torch.distributed``: NCCL on GPUs,
gloo in the CPU tests) and each rank merges the G records on the device
(``mc_merge_records``: max similarity, ties to the newer position, then the
threshold / k epilogue).  That all-gather of B x 32 bytes per rank is the
path's only collective.
* ``local_shards=G`` mode: one process drives all G shard rings (on
  ``devices``, one per shard; several shards may share a device).  Each
  shard's local scan writes its records straight into its slice of one
  [G, B] record buffer on the merging device (a peer copy when the shard lives
  on another GPU), and the merge runs there — no collective at all.  With
  every shard on one device this is the single-GPU test bed of the sharded
  kernels (tests/test_gpu_parity.py).

Partition: round-robin by append position (module doc above) keeps the
shards within one row of each other at every fill level and through age
evictions, so the slowest shard — which sets the lookup's time — never
holds more than ceil(n/G) rows.  A contiguous ring-slot range per shard
(SURVEY.md §8 e) balances only a full ring; DESIGN.md §7 quantifies the
difference on the C4 trace (profiles/partition_r02.txt).

FIFO bookkeeping evicts before it appends — the capacity evictions an insert
will cause are known up front — so a shard ring of ceil(C/G) rows never has
to displace anything on its own.
"""
from __future__ import annotations

import math
import os

import numpy as np

from .cache import _HIT, _EMPTY, _MISS_EMPTY, EntryFifo, _unit_norm, _default_device
from .records import (
    DEFAULT_DIM,
    LARGE,
    POLICIES,
    POLICY_ALL,
    POLICY_DISABLED,
    POLICY_LARGE,
    SMALL,
    CacheEntry,
    EmbeddingError,
    RetrievalResult,
    ThresholdTable,
    make_result,
)

RECORD_BYTES = 32  # sizeof(mc_record)
_NEED_RESCAN = 0x80  # MC_FLAG_NEED_RESCAN
_MERGE_SLOTS = 2  # MC_MERGE_SLOTS
_SLACK = 8  # PIPE_SLACK: rows a shard may append while a submitted lookup can still need its rescan


class _ShardedPending:
    """A submitted sharded lookup (ShardedSemanticCache.retrieve_async / retrieve_batch_async).
    Its records are gathered and its merge is enqueued at submit; ``result()`` reads the
    decisions (running the rescan round first if a shard's certificate failed) and returns what
    retrieve() / retrieve_batch() would have returned at submit time.  A later lookup, a bulk
    load or enough inserts complete it first, so a dropped future never wedges the cache."""

    __slots__ = ("_c", "_Q", "_slot", "_p0", "_rec", "_single", "_appended", "_done", "_error")

    def __init__(self, cache, Q, slot, p0, rec, single):
        self._c, self._Q, self._slot, self._p0, self._rec, self._single = cache, Q, slot, p0, rec, single
        self._appended = cache._appended
        self._done = self._error = None

    def _complete(self) -> None:
        c = self._c
        if c is None:
            return
        self._c = None
        try:
            c._pending.remove(self)
        except ValueError:
            pass
        try:
            gathered, stream, locals_ = self._rec
            live, sim, k, flags = c.ring.merge_wait(self._slot)
            if locals_ and (flags & _NEED_RESCAN).any():  # the same on every rank (SPMD)
                c._rescan(self._Q, gathered, stream, locals_)
                live, sim, k, flags = c.ring.merge_records(gathered, c.n_shards, self._Q.shape[0], self._p0, stream)
            at = c._store.at_position
            out = []
            for i, f in enumerate(np.asarray(flags).tolist()):
                if f & _HIT:
                    out.append(make_result(at(self._p0 + int(live[i])), float(sim[i]), int(k[i]) or None))
                elif f & _EMPTY:
                    out.append(_MISS_EMPTY)
                else:
                    out.append(make_result(None, float(sim[i]), None))
            self._done = out[0] if self._single else out
        except BaseException as exc:  # kept: result() re-raises it
            self._error = exc
        finally:
            c._store.unpin()

    def result(self):
        if self._c is not None:
            self._complete()
        if self._error is not None:
            raise self._error
        return self._done


def _count_owned(p_lo: int, n: int, g: int, G: int) -> int:
    """How many of the global positions p_lo .. p_lo+n-1 satisfy p % G == g."""
    if n <= 0:
        return 0
    first = p_lo + ((g - p_lo) % G)
    return 0 if first >= p_lo + n else 1 + (p_lo + n - 1 - first) // G


class ShardedSemanticCache:
    """SemanticCache API over G entry shards (one per rank of a process group).

    ``ring_factory(capacity, dim, device)`` builds the shard ring (default: the
    native ``DeviceRing``); ``comm`` defaults to ``torch.distributed``.
    """

    def __init__(self, capacity: int, dim: int = DEFAULT_DIM, policy: str = POLICY_ALL,
                 max_age_s: float | None = None, device: int | None = None, group=None,
                 ring_factory=None, local_shards: int | None = None, devices=None):
        if capacity < 1:
            raise ValueError(f"capacity must be >= 1, got {capacity}")
        if policy not in POLICIES:
            raise ValueError(f"unknown cache policy {policy!r}, expected one of {POLICIES}")
        if max_age_s is not None and max_age_s <= 0:
            raise ValueError(f"max_age_s must be positive, got {max_age_s}")
        self.capacity = int(capacity)
        self.dim = int(dim)
        self.policy = policy
        self.max_age_s = max_age_s
        self.device = _default_device() if device is None else int(device)
        self._group = group
        if local_shards is None:
            import torch.distributed as dist

            self._dist = dist
            self.n_shards = dist.get_world_size(group)
            self.shard = dist.get_rank(group)
            owned = {self.shard: self.device}
        else:
            if local_shards < 1:
                raise ValueError(f"local_shards must be >= 1, got {local_shards}")
            self._dist = None
            self.n_shards = int(local_shards)
            self.shard = 0
            devs = [self.device] * self.n_shards if devices is None else [int(x) for x in devices]
            if len(devs) != self.n_shards:
                raise ValueError(f"need one device per shard: {len(devs)} devices for {self.n_shards} shards")
            owned = dict(enumerate(devs))
        self._store = EntryFifo()
        self._next_seq = 0
        self._appended = 0  # global append position of the next entry
        if ring_factory is None:
            from ._native import DeviceRing as ring_factory
        cap_g = math.ceil(self.capacity / self.n_shards)
        self._rings = {}
        for g, dev in owned.items():
            ring = ring_factory(cap_g, self.dim, dev)
            ring.configure_shard(self.n_shards, g)
            self._rings[g] = ring
        self.ring = self._rings[min(self._rings)]  # the merging shard's ring
        self._table_key = None
        self._pending: list[_ShardedPending] = []  # submitted lookups, oldest first (at most two)

    # -- bookkeeping -------------------------------------------------------------
    def __len__(self) -> int:
        return len(self._store)

    def entries(self) -> list[CacheEntry]:
        return list(self._store)

    @property
    def next_seq(self) -> int:
        return self._next_seq

    @property
    def oldest_position(self) -> int:
        return self._appended - len(self._store)

    def admits(self, producer: str) -> bool:
        if self.policy == POLICY_DISABLED:
            return False
        if self.policy == POLICY_LARGE:
            return producer == LARGE
        return True

    def _evict(self, n: int, evicted: list) -> None:
        """Drop the n oldest entries everywhere; each owned shard drops the ones it holds."""
        if n <= 0:
            return
        p_lo = self.oldest_position
        for g, ring in self._rings.items():
            mine = _count_owned(p_lo, n, g, self.n_shards)
            if mine:
                ring.evict_front(mine)
        for _ in range(n):
            evicted.append(self._store.popleft())

    def insert(self, entry: CacheEntry) -> list[CacheEntry]:
        """cache.py:206-235 semantics, on every rank with the same entry stream."""
        if not self.admits(entry.producer):
            return []
        if entry.producer not in (LARGE, SMALL):
            raise ValueError(f"unknown producer {entry.producer!r}")
        emb = entry.embedding
        if emb.shape != (self.dim,):
            raise EmbeddingError(f"entry embedding has shape {emb.shape}, cache dim is {self.dim}")
        if not _unit_norm(emb):
            raise EmbeddingError(f"entry {entry.id!r} embedding is not unit norm")
        store = self._store
        if store and entry.seq <= store[-1].seq:
            raise ValueError(f"seq must increase: got {entry.seq} after {store[-1].seq}")
        if self._pending and self._appended - self._pending[0]._appended >= _SLACK:
            self._settle()  # a rescan of theirs must still find the window they scanned
        evicted: list[CacheEntry] = []
        if self.max_age_s is not None:
            horizon = entry.inserted_at - self.max_age_s
            n_age = 0
            for e in store:
                if e.inserted_at < horizon:
                    n_age += 1
                else:
                    break
            self._evict(n_age, evicted)
        # capacity eviction of the append below, applied first (see module doc)
        self._evict(len(store) + 1 - self.capacity, evicted)
        store.append(entry)
        ring = self._rings.get(self._appended % self.n_shards)
        if ring is not None:
            ring.append1(emb)
        self._appended += 1
        if entry.seq >= self._next_seq:
            self._next_seq = entry.seq + 1
        return evicted

    def add(self, id: str, embedding: np.ndarray, producer: str, inserted_at: float) -> list[CacheEntry]:
        return self.insert(CacheEntry(id, embedding, producer, self._next_seq, inserted_at))

    def bulk_load(self, entries) -> list[CacheEntry]:
        """insert() for every entry in order (same answers, errors and evictions on every rank),
        with one device append of this shard's rows; see SemanticCache.bulk_load."""
        from .cache import _validated_prefix

        entries = list(entries)
        self._settle()
        batch, bad = _validated_prefix(self, entries)
        if self.max_age_s is not None or len(batch) > self.capacity:  # the per-entry path decides evictions
            out: list[CacheEntry] = []
            for e in entries:
                out.extend(self.insert(e))
            return out
        evicted: list[CacheEntry] = []
        if batch:
            # capacity evictions first (module doc), then this shard's share of the appends
            self._evict(len(self._store) + len(batch) - self.capacity, evicted)
            p0 = self._appended
            for g, ring in self._rings.items():
                mine = [e.embedding for j, e in enumerate(batch) if (p0 + j) % self.n_shards == g]
                if mine:
                    ring.append(np.stack(mine))
            self._store.extend(batch)
            self._appended += len(batch)
            self._next_seq = max(self._next_seq, batch[-1].seq + 1)
        if bad is not None:
            self.insert(bad)  # raises the reference's error for the first invalid entry
        return evicted

    # -- lookups (SPMD: every rank passes the same queries) -----------------------
    def _comm_stream(self, dev):
        """A dedicated (non-default) stream for the record exchange and the merge: every
        shard's scan is ordered before it by an event (mc_retrieve_local_async), which a
        legacy default stream (handle 0, i.e. "the ring's own stream" to the C ABI) would not
        get."""
        import torch

        st = getattr(self, "_streams", None)
        if st is None:
            st = self._streams = {}
        if dev not in st:
            st[dev] = torch.cuda.Stream(dev) if dev.type == "cuda" else None
        return st[dev]

    def _records(self, Q: np.ndarray):
        """Every shard's local records -> one [G, B] record buffer on the merging device.

        Host-fed lookups take the scan without the exhaustive rescan behind it
        (mc_retrieve_local_submit); a record whose certificate failed comes back from the merge
        as MC_FLAG_NEED_RESCAN and ``_rescan`` runs the second round.  Returns the gathered
        buffer, the exchange stream and the per-shard record buffers (for that round)."""
        import contextlib

        import torch

        B = Q.shape[0]
        nb = B * RECORD_BYTES
        dev = self.ring.records_device()
        cs = self._comm_stream(dev)
        ctx = torch.cuda.stream(cs) if cs is not None else contextlib.nullcontext()
        sp = cs.cuda_stream if cs is not None else 0
        locals_ = []
        with ctx:
            gathered = torch.empty(self.n_shards * nb, dtype=torch.uint8, device=dev)
            if self._dist is not None:  # one shard per rank: all-gather the B records (the only collective)
                local = torch.empty(nb, dtype=torch.uint8, device=dev)
                G = self.n_shards
                split = G > 1 or os.environ.get("MC_SHARD_SPLIT_UPLOAD") == "1"  # (1: test the path at G = 1)
                if dev.type == "cuda" and split and B > 4 and B % G == 0 and self.dim % 64 == 0:
                    # the batch enters once: each rank uploads its 1/G of the rows and the ranks
                    # all-gather the queries over NVLink (mc_retrieve_local_device, rescan included)
                    part = B // G
                    mine = torch.from_numpy(Q[self.shard * part:(self.shard + 1) * part]).to(dev).reshape(-1)
                    full = torch.empty(B * self.dim, dtype=torch.float64, device=dev)
                    self._dist.all_gather_into_tensor(full, mine, group=self._group)
                    self.ring.retrieve_local_device(full, B, local, sp)
                else:
                    self.ring.retrieve_local_submit(Q, local, sp)
                    locals_.append((self.ring, local))
                self._dist.all_gather_into_tensor(gathered, local, group=self._group)
                return gathered, sp, locals_
            for g, ring in self._rings.items():  # every shard in this process: write the slices directly
                rdev = ring.records_device()
                if rdev == dev:
                    part = gathered[g * nb:(g + 1) * nb]
                    ring.retrieve_local_submit(Q, part, sp)
                    locals_.append((ring, part))
                else:  # shard on a peer GPU: its records cross NVLink as one peer copy
                    rs = self._comm_stream(rdev)
                    local = torch.empty(nb, dtype=torch.uint8, device=rdev)
                    ring.retrieve_local_submit(Q, local, rs.cuda_stream)
                    cs.wait_stream(rs)
                    gathered[g * nb:(g + 1) * nb].copy_(local, non_blocking=True)
                    local.record_stream(cs)
                    locals_.append((ring, local))
        return gathered, sp, locals_

    def _rescan(self, Q: np.ndarray, gathered, sp, locals_) -> None:
        """Second round after a merge reported MC_FLAG_NEED_RESCAN (the same on every rank: all
        ranks merged the same gathered records): each shard rescans the flagged queries
        exhaustively in float64, in place, and the records are gathered again."""
        import torch

        nb = Q.shape[0] * RECORD_BYTES
        dev = self.ring.records_device()
        cs = self._comm_stream(dev)
        with torch.cuda.stream(cs):
            if self._dist is not None:
                ring, local = locals_[0]
                ring.rescan_local(Q, local, sp)
                self._dist.all_gather_into_tensor(gathered, local, group=self._group)
                return
            for g, (ring, buf) in zip(sorted(self._rings), locals_):
                rdev = ring.records_device()
                if rdev == dev:
                    ring.rescan_local(Q, buf, sp)
                else:
                    rs = self._comm_stream(rdev)
                    rs.wait_stream(cs)
                    ring.rescan_local(Q, buf, rs.cuda_stream)
                    cs.wait_stream(rs)
                    gathered[g * nb:(g + 1) * nb].copy_(buf, non_blocking=True)
                    buf.record_stream(cs)

    def retrieve_batch(self, Q: np.ndarray, table: ThresholdTable) -> list[RetrievalResult]:
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        if Q.ndim != 2 or Q.shape[1] != self.dim:
            raise EmbeddingError(f"query batch has shape {Q.shape}, cache dim is {self.dim}")
        if Q.shape[0] == 0:
            return []
        self._settle()
        if not self._store:
            return [_MISS_EMPTY] * Q.shape[0]
        key = (table.pairs, table.total_steps)
        if key != self._table_key:
            for ring in self._rings.values():
                ring.set_table(table.pairs, table.total_steps)
            self._table_key = key
        gathered, stream, locals_ = self._records(Q)
        live, sim, k, flags = self.ring.merge_records(gathered, self.n_shards, Q.shape[0], self.oldest_position,
                                                      stream)
        if locals_ and (flags & _NEED_RESCAN).any():
            self._rescan(Q, gathered, stream, locals_)
            live, sim, k, flags = self.ring.merge_records(gathered, self.n_shards, Q.shape[0], self.oldest_position,
                                                          stream)
        at = self._store.live
        out = []
        for i, f in enumerate(np.asarray(flags).tolist()):
            if f & _HIT:
                out.append(make_result(at(int(live[i])), float(sim[i]), int(k[i]) or None))
            elif f & _EMPTY:
                out.append(_MISS_EMPTY)
            else:
                out.append(make_result(None, float(sim[i]), None))
        return out

    def retrieve(self, q: np.ndarray, table: ThresholdTable) -> RetrievalResult:
        if q.shape != (self.dim,):
            raise EmbeddingError(f"query has shape {q.shape}, cache dim is {self.dim}")
        return self.retrieve_batch(q[None, :], table)[0]

    # -- pipelined lookups ----------------------------------------------------------
    def _settle(self) -> None:
        """Complete the submitted lookups (their answers stay in their futures)."""
        while self._pending:
            self._pending[0]._complete()

    def _submit(self, Q: np.ndarray, table: ThresholdTable, single: bool):
        from .cache import _Ready

        if not self._store:
            return _Ready(_MISS_EMPTY if single else [_MISS_EMPTY] * Q.shape[0])
        key = (table.pairs, table.total_steps)
        if key != self._table_key:
            self._settle()  # a rescan round merges with the table of its submit
            for ring in self._rings.values():
                ring.set_table(table.pairs, table.total_steps)
            self._table_key = key
        if len(self._pending) >= _MERGE_SLOTS:
            self._pending[0]._complete()
        slot = min({0, 1} - {p._slot for p in self._pending})
        rec = self._records(Q)
        p0 = self.oldest_position
        self.ring.merge_submit(rec[0], self.n_shards, Q.shape[0], p0, rec[1], slot)
        self._store.pin()
        fut = _ShardedPending(self, Q, slot, p0, rec, single)
        self._pending.append(fut)
        return fut

    def retrieve_async(self, q: np.ndarray, table: ThresholdTable):
        """retrieve() split in two (SemanticCache.retrieve_async): the lookup is enqueued against
        the current cache and ``.result()`` returns what retrieve() would have returned then.
        Inserts may go on meanwhile; two lookups may be pending (the merge's two result slots)."""
        if q.shape != (self.dim,):
            raise EmbeddingError(f"query has shape {q.shape}, cache dim is {self.dim}")
        return self._submit(np.ascontiguousarray(q[None, :], dtype=np.float64), table, True)

    def retrieve_batch_async(self, Q: np.ndarray, table: ThresholdTable):
        """retrieve_batch() split in two, like retrieve_async."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        if Q.ndim != 2 or Q.shape[1] != self.dim:
            raise EmbeddingError(f"query batch has shape {Q.shape}, cache dim is {self.dim}")
        if Q.shape[0] == 0:
            from .cache import _Ready

            return _Ready([])
        return self._submit(Q, table, False)

    def shard_sizes(self) -> list[int]:
        """Live rows per shard held by this process (shard id order)."""
        return [len(self._rings[g]) for g in sorted(self._rings)]

    def close(self) -> None:
        self._settle()
        for ring in self._rings.values():
            ring.close()
