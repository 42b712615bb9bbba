"""Batched callers of the lookup: the reference's request intake, one
batched device lookup per burst of same-instant arrivals.

The reference classifies one request per ``cache.retrieve`` (``scheduler.classify``,
pkg/src/mixserve/scheduler.py:70-90), called once per arrival event
(``Simulation._on_arrival``, engine.py:201-209).  Requests that arrive at the same
instant all see the same cache state — nothing between two such arrivals mutates the
cache: completions at that instant are processed first (the event heap orders
(time, kind) with EVENT_COMPLETION < EVENT_ARRIVAL, engine.py:30-33) and dispatch only
reads it (the reclassification, engine.py:329-338) — so their lookups can be one
``retrieve_batch``, which runs on the tensor-core scan from B = 5 (one pass over the
ring for the whole burst instead of one per request).  The per-request side effects stay
exactly the reference's, in arrival order.
"""
from __future__ import annotations

import numpy as np

STATUS_QUEUED_HIT = "queued_hit"    # scheduler.py:13
STATUS_QUEUED_MISS = "queued_miss"  # scheduler.py:14


def _lookup_all(cache, Q: np.ndarray, table):
    batch = getattr(cache, "retrieve_batch", None)
    if batch is not None:
        return batch(Q, table)
    return [cache.retrieve(q, table) for q in Q]  # a cache without a batch API (the stock reference)


def apply_classification(r, result, queues):
    """What ``scheduler.classify`` does with its lookup's result (scheduler.py:79-89)."""
    r.similarity = result.similarity
    if result.hit:
        r.k = result.k
        r.source_entry_id = result.entry.id
        r.source_embedding = result.entry.embedding
        r.source_age_s = r.arrival_time - result.entry.inserted_at
        r._advance(STATUS_QUEUED_HIT)
        queues.hit.append(r)
    else:
        r._advance(STATUS_QUEUED_MISS)
        queues.miss.append(r)
    return r


def lookup_requests(requests, cache, table):
    """One batched lookup for the requests' query embeddings (their classify() lookups)."""
    Q = np.stack([np.asarray(r.query_embedding, dtype=np.float64) for r in requests])
    return _lookup_all(cache, Q, table)


def classify_batch(requests, cache, table, queues):
    """``scheduler.classify`` for every request of `requests` (same arrival instant), with one
    batched lookup; returns the requests.  Field updates and queue order as classify
    (scheduler.py:78-89) applied to each request in turn."""
    requests = list(requests)
    if requests:
        for r, result in zip(requests, lookup_requests(requests, cache, table)):
            apply_classification(r, result, queues)
    return requests


def install_batched_arrivals(sim, engine_module):
    """Make a reference ``Simulation`` classify each burst of same-instant arrivals with one
    batched lookup.  `engine_module` is ``mixserve.engine`` (for its event kinds and Request).

    The replacement pops the burst's remaining arrival events off the heap and looks the whole
    burst up at once; then, for each request in arrival order, it applies that request's
    classification and runs the original per-arrival bookkeeping and dispatch
    (engine.py:201-209) — so each dispatch sees exactly the queues it sees in the reference."""
    import heapq

    arrival = engine_module.EVENT_ARRIVAL
    Request = engine_module.Request
    stats = {"bursts": 0, "batched_lookups": 0}

    def on_arrival(rec):
        burst = [rec]
        heap = sim._heap
        while heap and heap[0][0] == sim.clock and heap[0][1] == arrival:
            burst.append(heapq.heappop(heap)[3])
        reqs = [Request(x.id, sim.clock, x.embedding) for x in burst]
        results = lookup_requests(reqs, sim.cache, sim.table)
        stats["bursts"] += 1
        stats["batched_lookups"] += len(reqs) if len(reqs) > 1 else 0
        for r, result in zip(reqs, results):  # engine.py:201-209, per request
            sim._arrivals_pending -= 1
            apply_classification(r, result, sim.queues)
            sim._period_arrivals += 1
            if r.is_hit:
                sim._period_hits += 1
                sim._period_k[r.k] = sim._period_k.get(r.k, 0) + 1
            sim._dispatch_idle()

    sim._on_arrival = on_arrival
    return stats
