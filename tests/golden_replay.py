"""Replay helper for the golden op logs written by tests/golden/make_golden.py."""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
SCENARIOS = sorted(p.stem for p in GOLDEN.glob("*.npz"))
PRODUCER = {0: "large", 1: "small"}


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        g = {k: z[k] for k in z.files}
    g["policy"] = str(g["policy"])
    age = float(g["max_age_s"])
    g["max_age_s"] = None if math.isnan(age) else age
    g["pairs"] = tuple((int(k), float(t)) for k, t in zip(g["ks"], g["taus"]))
    return g


def replay(g: dict, make_cache, make_entry, make_table, retrieve):
    """Drive a cache through the op log; returns list of (live, seq, sim, k) per retrieve.

    ``retrieve(cache, q, table)`` returns (entry_seq | None, live | None, sim | None, k | None).
    """
    cache = make_cache(int(g["capacity"]), int(g["dim"]), g["policy"], g["max_age_s"])
    table = make_table(g["pairs"], int(g["total_steps"]))
    out = []
    for i, kind in enumerate(g["kind"]):
        v = g["vec"][i]
        if kind == 0:
            seq = int(g["seq"][i])
            ev = cache.insert(make_entry(f"e{seq}", v.copy(), PRODUCER[int(g["prod"][i])], seq, float(g["t"][i])))
            assert len(ev) == int(g["n_evicted"][i]), (i, len(ev), g["n_evicted"][i])
            assert len(cache) == int(g["size_after"][i])
        else:
            out.append(retrieve(cache, v.copy(), table))
    return out


def expected(g: dict):
    m = g["kind"] == 1
    seqs = g["r_seq"][m]
    lives = g["r_live"][m]
    sims = g["r_sim"][m]
    ks = g["r_k"][m]
    return [
        (None if s < 0 else int(s), None if l < 0 else int(l), None if math.isnan(x) else float(x), None if k < 0 else int(k))
        for s, l, x, k in zip(seqs, lives, sims, ks)
    ]
