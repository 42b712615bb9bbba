"""Replay test_random_operation_sequences_every_path[seed] and report the first mismatch in detail."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.retrieval import OracleCache, OracleEntry, OracleTable  # noqa: E402
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable, _native  # noqa: E402

seed = int(sys.argv[1])
rng = np.random.default_rng(1000 + seed)
dim = int(rng.choice([8, 96, 200, 512, 768, 1000]))
cap = int(rng.integers(50, 3000))
age = float(rng.choice([0.0, 400.0]))
paths = [_native.PATH_AUTO, _native.PATH_STREAM8, _native.PATH_GEMV8, _native.PATH_GEMV, _native.PATH_GEMM,
         _native.PATH_GEMM8]
print("dim", dim, "cap", cap, "age", age)
c = SemanticCache(capacity=cap, dim=dim, policy="all", max_age_s=age or None)
o = OracleCache(cap, dim, max_age_s=age or None)
table, ot = ThresholdTable.default(), OracleTable()
centers = rng.standard_normal((6, dim))
t, seq = 0.0, 0


def fresh(n):
    global t, seq
    out = []
    for _ in range(n):
        v = centers[rng.integers(0, 6)] + 1.2 * rng.standard_normal(dim) / np.sqrt(max(dim, 1)) * 4
        t += float(rng.exponential(1.0))
        out.append(CacheEntry(f"e{seq}", v / np.linalg.norm(v), "large" if rng.random() < 0.8 else "small", seq, t))
        seq += 1
    return out


def consistent(tag):
    if not o.meta:
        return
    M = np.stack([m.embedding for m in o.meta])
    c.ring.set_path(2)
    l2, s2, k2, f2 = c.retrieve_flags(M, table)
    bad = [j for j in range(len(M)) if abs(s2[j] - 1.0) > 1e-9]
    if bad:
        j = bad[0]
        print("INCONSISTENT after", tag, ": live", j, "of", len(M), "(", o.meta[j].id, ") best", int(l2[j]), float(s2[j]),
              "n bad", len(bad), "first bad ids", [o.meta[b].id for b in bad[:5]])
        for pth in (2, 2, 1, 6, 5):
            c.ring.set_path(pth)
            l3, s3, k3, f3 = c.retrieve_flags(M, table)
            print("  recheck path", pth, "bad:", [j2 for j2 in range(len(M)) if abs(s3[j2] - 1.0) > 1e-9][:6])
        hid = [e.id for e in c.entries()]
        oid = [m.id for m in o.meta]
        print(" host FIFO == oracle:", hid == oid, "len host", len(hid), "len oracle", len(oid), "ring", len(c.ring))
        if hid != oid:
            d = next(i for i in range(min(len(hid), len(oid))) if hid[i] != oid[i])
            print(" first difference at", d, hid[d - 2:d + 3], oid[d - 2:d + 3])
        for b in bad[:3]:
            rows3 = c.ring.debug_read_row(b)
            for nm, rr in zip(("f64", "f16", "i8"), rows3):
                dd = M @ rr
                print("   copy", nm, "at live", b, "best match", o.meta[int(np.argmax(dd))].id, float(dd.max()))
            row = rows3[0]
            dots = M @ row
            print("  device row at live", b, "is oracle entry", o.meta[int(np.argmax(dots))].id, "dot", float(dots.max()),
                  "| matches any evicted?", "norm", float(np.linalg.norm(row)))
        print(" self-hit index for bad rows:", [(b, int(l2[b])) for b in bad], " neighbours:",
              [(b, int(l2[b])) for b in range(max(0, bad[0] - 3), min(len(M), bad[-1] + 4))])
        sys.exit(2)


for step in range(60):
    op = rng.random()
    if op < 0.35:
        fr = fresh(int(rng.integers(1, 40)))
        for e in fr:
            c.insert(e)
            o.insert(OracleEntry(e.id, e.embedding, e.producer, e.seq, e.inserted_at))
        consistent(f"step {step}: {len(fr)} inserts (n_live {len(o.meta)})")
    elif op < 0.45:
        batch = fresh(int(rng.integers(1, 400)))
        if step == 36:
            for j, e in enumerate(batch):
                h0 = len(o.meta)
                ev = c.insert(e)
                o.insert(OracleEntry(e.id, e.embedding, e.producer, e.seq, e.inserted_at))
                print("  insert", j, e.id, "evicted", len(ev), "n_live", len(o.meta), "pending?")
                if j in (15, 16, 17, 18, 19, 20) or j % 20 == 0:
                    consistent(f"step 36 insert {j}")
        else:
            c.bulk_load(batch)
            for e in batch:
                o.insert(OracleEntry(e.id, e.embedding, e.producer, e.seq, e.inserted_at))
        consistent(f"step {step}: bulk {len(batch)} (n_live {len(o.meta)})")
    else:
        path = int(rng.choice(paths))
        c.ring.set_path(path)
        B = int(rng.choice([1, 1, 2, 3, 4, 5, 17, 130]))
        Q = centers[rng.integers(0, 6, B)] + 1.2 * rng.standard_normal((B, dim)) / np.sqrt(dim) * 4
        Q /= np.linalg.norm(Q, axis=1, keepdims=True)
        use_async = B == 1 and rng.random() < 0.5
        print("step", step, "lookup path", path, "B", B, "async", use_async, "n_live", len(o.meta))
        if use_async:
            got = [c.retrieve_async(Q[0], table).result()]
        else:
            got = c.retrieve_batch(Q, table)
        if not o.meta:
            continue
        live, sim, k, flags = c.retrieve_flags(Q, table)
        M = np.stack([m.embedding for m in o.meta])
        for i, (q, r) in enumerate(zip(Q, got)):
            e, s, kk = o.retrieve_entry(q, ot)
            if (r.entry.id if r.hit else None) != (e.id if e is not None else None) or r.k != kk:
                sims = M @ q
                order = np.argsort(-sims)[:6]
                print("MISMATCH step", step, "path", path, "B", B, "async", use_async, "query", i)
                print(" got", r.entry.id if r.hit else None, r.similarity, r.k, " want", e.id if e else None, s, kk)
                print(" flags (retrieve_flags)", hex(int(flags[i])), "live", live[i], "sim", sim[i])
                print(" oracle top:", [(o.meta[j].id, float(sims[j])) for j in order])
                print(" n live", len(o.meta), "ring", len(c.ring), "stats", c.ring.stats())
                want_live = [m.id for m in o.meta].index(e.id)
                print(" want live index", want_live, "of", len(o.meta))
                for name, pth in (("gemv", 1), ("gemv8", 5), ("stream8", 6), ("gemm", 2), ("gemm1", 3), ("gemm8", 7)):
                    c.ring.set_path(pth)
                    l2, s2, k2, f2 = c.retrieve_flags(Q, table)
                    print("   ", name, "live", int(l2[i]), "sim", float(s2[i]), "flags", hex(int(f2[i])))
                sys.exit(1)
print("no mismatch")
