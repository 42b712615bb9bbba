"""Record the cache traffic of REAL reference Simulation runs as golden op logs.

Run from the repo root in the build container (where /root/reference exists):

    python tests/golden/make_sim_golden.py

For each shipped config (pkg/configs/*.cfg) the reference's own trace
generator (workload.py:141-142) and Simulation (engine.py:108-338) run with
``mixserve.cache.SemanticCache`` swapped for a recording subclass.  Every
``insert`` (scheduler.on_completion -> add, engine.py:244-249) and every
``retrieve`` (scheduler.classify, scheduler.py:78; the dispatch-time
reclassification, engine.py:329-338) is logged with its inputs and the
reference's answer, in make_golden.py's op-log format (tests/golden/sim_*.npz).
The Simulation is deterministic given the cache's answers, so a cache that
reproduces every logged answer — the GPU path, replayed by
tests/test_gpu_parity.py::test_golden_op_logs — drives the reference control
plane through the identical trajectory.  The run's report is kept too
(sim_reports.json) for the live drop-in check in tests/test_dropin_reference.py.
"""
from __future__ import annotations

import dataclasses
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import mixserve.cache as mc  # noqa: E402
import mixserve.config as mconfig  # noqa: E402
from mixserve.config import load_sim_config  # noqa: E402
from mixserve.engine import run_simulation  # noqa: E402
from mixserve.workload import generate_trace  # noqa: E402

from make_golden import OP_INSERT, OP_RETRIEVE, OUT, PROD, Log  # noqa: E402

_Stock = mc.SemanticCache


class RecordingCache(_Stock):
    """The reference cache, logging every insert / retrieve into `log` (a make_golden.Log)."""

    log: Log | None = None

    def insert(self, entry):
        ev = super().insert(entry)
        g = self.log
        g.kind.append(OP_INSERT); g.vec.append(np.asarray(entry.embedding, dtype=np.float64).copy())
        g.prod.append(PROD[entry.producer]); g.seq.append(entry.seq); g.t.append(float(entry.inserted_at))
        g.r_seq.append(-1); g.r_live.append(-1); g.r_sim.append(np.nan); g.r_k.append(-1)
        g.n_evicted.append(len(ev)); g.size_after.append(len(self))
        return ev

    def retrieve(self, q, table):
        res = super().retrieve(q, table)
        g = self.log
        g.table = table
        g.kind.append(OP_RETRIEVE); g.vec.append(np.asarray(q, dtype=np.float64).copy())
        g.prod.append(-1); g.seq.append(-1); g.t.append(np.nan)
        if res.hit:
            g.r_seq.append(res.entry.seq)
            g.r_live.append([e.seq for e in self.entries()].index(res.entry.seq))
        else:
            g.r_seq.append(-1); g.r_live.append(-1)
        g.r_sim.append(np.nan if res.similarity is None else res.similarity)
        g.r_k.append(-1 if res.k is None else res.k)
        g.n_evicted.append(0); g.size_after.append(len(self))
        return res


def report_dict(result) -> dict:
    return json.loads(json.dumps(dataclasses.asdict(result.report), default=str))


def main():
    reports = {}
    for path in sorted((REF / "configs").glob("*.cfg")):
        cfg = load_sim_config(path)
        trace = generate_trace(cfg.workload)
        name = f"sim_{path.stem}"
        log = Log.__new__(Log)
        log.name = name
        log.meta = dict(capacity=cfg.cache_capacity, dim=cfg.cache_dim, policy=cfg.cache_policy,
                        max_age_s=np.nan if cfg.cache_max_age_s is None else cfg.cache_max_age_s,
                        total_steps=cfg.threshold_table().total_steps)
        log.table = cfg.threshold_table()
        log.kind, log.vec, log.prod, log.seq, log.t = [], [], [], [], []
        log.r_seq, log.r_live, log.r_sim, log.r_k, log.n_evicted, log.size_after = [], [], [], [], [], []
        RecordingCache.log = log
        mc.SemanticCache = mconfig.SemanticCache = RecordingCache
        try:
            result = run_simulation(cfg, trace)
        finally:
            mc.SemanticCache = mconfig.SemanticCache = _Stock
        reports[path.stem] = {"n_trace": len(trace), "report": report_dict(result),
                              "audit_sha": _sha(result.audit)}
        if log.kind:
            log.save()
        else:
            print(f"{name}: no cache traffic (policy {cfg.cache_policy!r}); nothing to replay")
    (OUT / "sim_reports.json").write_text(json.dumps(reports, sort_keys=True, indent=1) + "\n")


def _sha(rows) -> str:
    import hashlib

    return hashlib.sha256(json.dumps(rows, sort_keys=True, default=str).encode()).hexdigest()


if __name__ == "__main__":
    main()
