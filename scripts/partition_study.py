"""Shard balance of the two partitions on C4-style traces (host-only study).

A lookup's time on G GPUs is set by the slowest shard: each scans its own live rows (HBM-bound,
~0.12 ns per 768-dim row at the measured 6.5 TB/s, bench.py single_gpu_large) and the merge
waits for all.  Compared for one FIFO of capacity C:
  * round-robin by append position (this build): shard g holds positions p = g (mod G);
  * contiguous ring-slot ranges (SURVEY.md §8 e): slot s = p mod C lives on GPU floor(s / ceil(C/G)).
Traces: the fill from empty, the capacity-bound steady state (the window wraps), and an
age-bound steady state (reference max_age_s eviction, cache.py:226-229) holding ~60 % of C.

    python scripts/partition_study.py   ->  profiles/partition_r02.txt
"""
import math
from pathlib import Path

import numpy as np

C = 1_000_000
NS_PER_ROW = 0.119e-3 / 1e6 * 1e9  # bench.py c4_b1: 0.119 ms per 1M-row B=1 lookup on one GPU


def loads(p0, n, G):
    """Live positions [p0, p0 + n): rows per shard under both partitions."""
    rr = np.array([(n - ((g - p0) % G) + G - 1) // G if n > ((g - p0) % G) else 0 for g in range(G)])
    cg = math.ceil(C / G)
    s0 = p0 % C
    cont = np.zeros(G, dtype=np.int64)
    # the window of n slots starting at s0 wraps at C at most once
    for a, b in ((s0, min(C, s0 + n)), (0, max(0, s0 + n - C))):
        for g in range(G):
            lo, hi = g * cg, min(C, (g + 1) * cg)
            cont[g] += max(0, min(b, hi) - max(a, lo))
    return rr, cont


rng = np.random.default_rng(7)
lines = [__doc__.strip().splitlines()[0], "", f"C = {C:,} rows; scan cost {NS_PER_ROW:.3f} ns/row (measured)", ""]
lines.append(f"{'trace':34s} {'G':>2s} {'live n':>9s} {'max shard RR':>13s} {'max shard range':>16s} "
             f"{'range/RR':>9s} {'slowest shard us RR / range':>28s}")
for G in (2, 4, 8):
    cases = []
    for n in (C // 100, C // 10, C // 2):  # fill from empty: the window starts at slot 0
        cases.append((f"fill, n = {n:,}", 0, n))
    for _ in range(3):  # capacity-bound steady state: full window at a random head
        cases.append(("full ring, random head", int(rng.integers(C, 10 * C)), C))
    for _ in range(3):  # age-bound steady state: ~60 % of C live, sliding head
        cases.append(("age-bound (0.6 C), random head", int(rng.integers(C, 10 * C)), int(0.6 * C)))
    for name, p0, n in cases:
        rr, cont = loads(p0, n, G)
        lines.append(f"{name:34s} {G:2d} {n:9,d} {rr.max():13,d} {cont.max():16,d} {cont.max() / rr.max():9.2f} "
                     f"{rr.max() * NS_PER_ROW / 1e3:13.1f} / {cont.max() * NS_PER_ROW / 1e3:6.1f}")
lines += ["", "Round-robin keeps every shard within one row of n/G at every fill level, through capacity and",
          "age eviction; contiguous slot ranges balance only a full ring, and while the cache fills or when",
          "age eviction keeps it partly empty the slowest GPU scans up to G x (fill) or ~1.7 x (0.6 C) the",
          "rows of a balanced shard.  Both partitions send each insert to exactly one GPU and need the same",
          "one all-gather of B x 32-byte records per lookup."]
out = Path(__file__).resolve().parents[1] / "profiles" / "partition_r02.txt"
out.write_text("\n".join(lines) + "\n")
print("\n".join(lines))
