"""Debug: replay test_random_operations_with_pending_lookups(seed) and dump the first mismatch."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import tests.test_gpu_parity as T  # noqa: E402

orig = T._close
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 9
try:
    T.test_random_operations_with_pending_lookups(seed)
    print("passed")
except AssertionError as exc:
    import traceback
    tb = traceback.extract_tb(exc.__traceback__)
    print("FAILED at", tb[-1].lineno, str(exc)[:300])
    frame = exc.__traceback__
    while frame.tb_next:
        frame = frame.tb_next
    loc = frame.tb_frame.f_locals
    r, want = loc.get("r"), loc.get("want")
    print("got", r.entry.id if r.hit else None, r.entry.seq if r.hit else None, r.similarity, r.k)
    e, sim, k = want
    print("want", e.id if e is not None else None, e.seq if e is not None else None, sim, k)
    up = frame.tb_frame.f_back.f_locals if frame.tb_frame.f_back else {}
    c = up.get("c")
    if c is not None:
        ents = c.entries()
        ids = [x.id for x in ents]
        print("len", len(c), "ring", len(c.ring), "first", ids[:3], "last", ids[-5:])
        bad = [(x.id, x.seq) for x in ents if x.id != f"e{x.seq}"]
        print("id/seq mismatches in the store:", bad[:10])
        q = up.get("q")
