"""Generate golden op logs by running the REAL reference (mixserve) in this container.

Run from the repo root in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Each scenario is a seeded sequence of ``insert`` / ``retrieve`` operations
applied to ``mixserve.cache.SemanticCache`` (cache.py:133-302).  The op log
(inputs) and the reference's answers (outputs) are written to
``tests/golden/<scenario>.npz`` so that the GPU box — which has no
/root/reference — can replay them against the CUDA path, and so that the CPU
oracle can be pinned against them.

Scenarios follow the reference's own tests / generators:
  kat_threshold      test_scheduler.py:20-22,47-60 (exact 2-d similarities)
  kat_tie            test_cache.py:212-222 (duplicate rows -> newest)
  kat_stale          test_engine.py:148-169 (similarity 0.26 -> k=10)
  churn_d6           test_cache.py:224-236 (seed 9, cap 50, D=6, max_age 200)
  churn_large_d16    policy "large" + capacity churn (test_cache.py:162-172 style)
  iid_d32            test_acceptance.py:411-443, scaled down (seed 4242)
  clustered_d64      workload.py gen_queries + image_embedding (engine.py:249)
  clustered_d768     same generators at the config-2 dimension
  duplicates_d16     exact duplicates through ring wrap-around (beta = 1)
  near_threshold_d48 q = s e + sqrt(1-s^2) u, s in {tau, tau +- 1e-9, tau +- 1e-12}
  nirvana_d32        nirvana-emulation.cfg:24 threshold table
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from mixserve.cache import CacheEntry, SemanticCache, ThresholdTable, normalize  # noqa: E402
from mixserve.workload import (  # noqa: E402
    GeneratorConfig,
    gen_arrivals,
    gen_queries,
    image_embedding,
)

OUT = Path(__file__).resolve().parent
OP_INSERT, OP_RETRIEVE = 0, 1
PROD = {"large": 0, "small": 1}
NIRVANA = ((5, 0.45), (10, 0.47), (15, 0.49), (20, 0.51), (25, 0.53), (30, 0.55))


class Log:
    def __init__(self, name, capacity, dim, policy="all", max_age_s=None, pairs=None, total_steps=50):
        self.name = name
        self.cache = SemanticCache(capacity=capacity, dim=dim, policy=policy, max_age_s=max_age_s)
        self.table = ThresholdTable(pairs, total_steps) if pairs else ThresholdTable.default(total_steps)
        self.meta = dict(capacity=capacity, dim=dim, policy=policy,
                         max_age_s=np.nan if max_age_s is None else max_age_s,
                         total_steps=total_steps)
        self.kind, self.vec, self.prod, self.seq, self.t = [], [], [], [], []
        self.r_seq, self.r_live, self.r_sim, self.r_k, self.n_evicted, self.size_after = [], [], [], [], [], []

    def insert(self, emb, producer="large", t=0.0, seq=None):
        seq = self.cache.next_seq if seq is None else seq
        ev = self.cache.insert(CacheEntry(f"e{seq}", emb, producer, seq, float(t)))
        self.kind.append(OP_INSERT); self.vec.append(np.asarray(emb, dtype=np.float64))
        self.prod.append(PROD[producer]); self.seq.append(seq); self.t.append(float(t))
        self.r_seq.append(-1); self.r_live.append(-1); self.r_sim.append(np.nan); self.r_k.append(-1)
        self.n_evicted.append(len(ev)); self.size_after.append(len(self.cache))

    def retrieve(self, q):
        res = self.cache.retrieve(q, self.table)
        self.kind.append(OP_RETRIEVE); self.vec.append(np.asarray(q, dtype=np.float64))
        self.prod.append(-1); self.seq.append(-1); self.t.append(np.nan)
        if res.hit:
            live = [e.seq for e in self.cache.entries()].index(res.entry.seq)
            self.r_seq.append(res.entry.seq); self.r_live.append(live)
        else:
            self.r_seq.append(-1); self.r_live.append(-1)
        self.r_sim.append(np.nan if res.similarity is None else res.similarity)
        self.r_k.append(-1 if res.k is None else res.k)
        self.n_evicted.append(0); self.size_after.append(len(self.cache))

    def save(self):
        ks = np.array([k for k, _ in self.table.pairs], dtype=np.int32)
        taus = np.array([t for _, t in self.table.pairs], dtype=np.float64)
        np.savez_compressed(
            OUT / f"{self.name}.npz",
            capacity=self.meta["capacity"], dim=self.meta["dim"], policy=self.meta["policy"],
            max_age_s=self.meta["max_age_s"], total_steps=self.meta["total_steps"],
            ks=ks, taus=taus,
            kind=np.array(self.kind, dtype=np.int8), vec=np.stack(self.vec),
            prod=np.array(self.prod, dtype=np.int8), seq=np.array(self.seq, dtype=np.int64),
            t=np.array(self.t, dtype=np.float64),
            r_seq=np.array(self.r_seq, dtype=np.int64), r_live=np.array(self.r_live, dtype=np.int64),
            r_sim=np.array(self.r_sim, dtype=np.float64), r_k=np.array(self.r_k, dtype=np.int32),
            n_evicted=np.array(self.n_evicted, dtype=np.int32),
            size_after=np.array(self.size_after, dtype=np.int64),
        )
        n_r = sum(1 for k in self.kind if k == OP_RETRIEVE)
        hits = sum(1 for s in self.r_seq if s >= 0)
        print(f"{self.name}: {len(self.kind)} ops, {n_r} retrieves, {hits} hits")


def unit(rng, d):
    return normalize(rng.standard_normal(d))


def exact_sim_query(s):
    return np.array([s, math.sqrt(1.0 - s * s)])


def kat_threshold():
    g = Log("kat_threshold", capacity=8, dim=2)
    g.retrieve(exact_sim_query(0.31))  # empty cache
    g.insert(np.array([1.0, 0.0]), t=0.0)
    for s in (0.31, 0.25, 0.29, 0.2499999, 0.26, 0.24, 0.305, 0.265, 1.0, -1.0, 0.0, 0.27, 0.28, 0.30):
        g.retrieve(exact_sim_query(s))
    g.save()


def kat_tie():
    g = Log("kat_tie", capacity=8, dim=4)
    emb = normalize([1.0, 1.0, 0.0, 0.0])
    g.insert(emb.copy(), t=0.0)
    g.insert(unit(np.random.default_rng(8), 4), t=1.0)
    g.insert(emb.copy(), t=2.0)
    g.retrieve(emb)
    g.retrieve(normalize([1.0, 0.9, 0.1, 0.0]))
    g.save()


def kat_stale():
    g = Log("kat_stale", capacity=100, dim=4)
    stale = normalize([0.26, np.sqrt(1 - 0.26 ** 2), 0.0, 0.0])
    e0 = np.array([1.0, 0.0, 0.0, 0.0])
    g.insert(stale, t=0.0)
    g.retrieve(e0)
    g.insert(e0.copy(), t=10.0)
    g.retrieve(e0)
    g.save()


def churn_d6():
    rng = np.random.default_rng(9)
    g = Log("churn_d6", capacity=50, dim=6, max_age_s=200.0)
    for i in range(300):
        g.insert(unit(rng, 6), producer=("large" if i % 3 else "small"), t=float(i), seq=i)
        if i % 2 == 0:
            g.retrieve(unit(rng, 6))
    g.save()


def churn_large_d16():
    rng = np.random.default_rng(21)
    g = Log("churn_large_d16", capacity=37, dim=16, policy="large", max_age_s=90.0)
    t = 0.0
    for i in range(600):
        t += float(rng.exponential(1.0))
        g.insert(unit(rng, 16), producer=("large" if rng.random() < 0.6 else "small"), t=t, seq=i)
        q = unit(rng, 16)
        if rng.random() < 0.3 and len(g.cache):
            e = g.cache.entries()[int(rng.integers(len(g.cache)))].embedding
            q = normalize(e + 0.9 * rng.standard_normal(16) / 4.0)
        g.retrieve(q)
    g.save()


def iid_d32():
    rng = np.random.default_rng(4242)
    g = Log("iid_d32", capacity=2000, dim=32)
    for i in range(2000):
        g.insert(normalize(rng.standard_normal(32)), t=float(i), seq=i)
    for _ in range(500):
        g.retrieve(normalize(rng.standard_normal(32)))
    g.save()


def clustered(name, dim, capacity, n_records, n_clusters, beta, seed=17, rate=60.0):
    spread = 0.0554 * math.sqrt(384.0 / dim)
    cfg = GeneratorConfig(rate_schedule=[(3600.0 * 10, rate)], n_clusters=n_clusters,
                          cluster_lifetime_s=600.0, spread=spread, beta=beta, dim=dim, seed=seed)
    arrivals = gen_arrivals(cfg)[:n_records]
    recs = gen_queries(cfg, arrivals)
    rng_img = np.random.default_rng([seed, 3])  # engine.py:35,119 IMAGE_STREAM
    g = Log(name, capacity=capacity, dim=dim)
    for r in recs:
        g.retrieve(r.embedding)
        g.insert(image_embedding(r.embedding, beta, rng_img), producer="large", t=r.arrival_ms / 1000.0)
    g.save()


def duplicates_d16():
    rng = np.random.default_rng(5)
    pool = [unit(rng, 16) for _ in range(10)]
    g = Log("duplicates_d16", capacity=64, dim=16)
    for i in range(400):
        g.insert(pool[int(rng.integers(10))].copy(), t=float(i))
        if i % 3 == 0:
            if rng.random() < 0.7:
                g.retrieve(pool[int(rng.integers(10))].copy())
            else:
                g.retrieve(unit(rng, 16))
    g.save()


def near_threshold_d48():
    rng = np.random.default_rng(48)
    g = Log("near_threshold_d48", capacity=200, dim=48)
    bases = [unit(rng, 48) for _ in range(200)]
    for i, b in enumerate(bases):
        g.insert(b, t=float(i))
    taus = [t for _, t in g.table.pairs]
    for j in range(160):
        e = bases[int(rng.integers(200))]
        u = rng.standard_normal(48)
        u -= (u @ e) * e
        u /= np.linalg.norm(u)
        tau = taus[j % len(taus)]
        s = tau + (0.0, 1e-9, -1e-9, 1e-12, -1e-12, 2e-16, -2e-16, 1e-6)[j % 8]
        g.retrieve(s * e + math.sqrt(1.0 - s * s) * u)
    g.save()


def nirvana_d32():
    rng = np.random.default_rng(77)
    g = Log("nirvana_d32", capacity=300, dim=32, pairs=NIRVANA)
    for i in range(300):
        g.insert(unit(rng, 32), t=float(i))
    for _ in range(200):
        e = g.cache.entries()[int(rng.integers(300))].embedding
        g.retrieve(normalize(e + rng.uniform(0.1, 0.4) * rng.standard_normal(32)))
    g.save()


if __name__ == "__main__":
    kat_threshold()
    kat_tie()
    kat_stale()
    churn_d6()
    churn_large_d16()
    iid_d32()
    # betas calibrated with calibrate_beta(0.311) at these dims, seed 17 (SURVEY.md §8 d)
    clustered("clustered_d64", dim=64, capacity=500, n_records=1500, n_clusters=24, beta=0.95)
    clustered("clustered_d768", dim=768, capacity=120, n_records=160, n_clusters=6, beta=0.962890625)
    duplicates_d16()
    near_threshold_d48()
    nirvana_d32()
