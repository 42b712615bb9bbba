"""Localise wrong small-batch answers: i.i.d. unit rows (seed 4242) at several dims, 10k entries,
each query through retrieve() (parameter-block path) and retrieve_flags (envelope path) and each
forced path, compared with the exact float64 argmax (newest among ties).  Diagnostic only."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
NQ = 300
for dim in (32, 64, 96, 128, 160, 256, 384, 768):
    for load in ("insert", "bulk"):
        rng = np.random.default_rng(4242)
        M = rng.standard_normal((N, dim))
        M /= np.linalg.norm(M, axis=1, keepdims=True)
        cache = SemanticCache(capacity=N, dim=dim)
        ents = [CacheEntry(f"e{i}", M[i], "large", i, float(i)) for i in range(N)]
        if load == "insert":
            for e in ents:
                cache.insert(e)
        else:
            cache.bulk_load(ents)
        table = ThresholdTable.default()
        Q = rng.standard_normal((NQ, dim))
        Q /= np.linalg.norm(Q, axis=1, keepdims=True)
        S = M @ Q.T
        want = S.argmax(axis=0)
        bad = {"retrieve": 0, "flags": 0, "stream8": 0, "gemv": 0}
        for t in range(NQ):
            q = Q[t]
            top = S[:, t].max()
            if (S[:, t] >= top - 1e-12).sum() > 1:
                continue
            r = cache.retrieve(q, table)
            live, sim, k, fl = cache.retrieve_flags(q[None], table)
            if int(live[0]) != want[t]:
                bad["flags"] += 1
            if r.hit and int(r.entry.id[1:]) != want[t]:
                bad["retrieve"] += 1
        for path, code in (("stream8", 6), ("gemv", 1)):
            cache.ring.set_path(code)
            for t in range(NQ):
                live, sim, k, fl = cache.retrieve_flags(Q[t][None], table)
                if int(live[0]) != want[t] and (S[:, t] >= S[:, t].max() - 1e-12).sum() == 1:
                    bad[path] += 1
            cache.ring.set_path(0)
        print(f"dim {dim:4d} N {N} load {load:6s} wrong/{NQ}: {bad}  stats {cache.ring.stats()}", flush=True)
        cache.close()
