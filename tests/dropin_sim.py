"""Run the reference Simulation on its shipped configs with the GPU drop-in installed
(test infrastructure for tests/test_dropin_reference.py; needs baseline/_ref from
scripts/stage_reference.sh).  Prints one JSON object: per config, whether the report and
the request audit equal the reference run recorded in tests/golden/sim_reports.json."""
import dataclasses
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "baseline" / "_ref")]

import mixserve.cache as mc  # noqa: E402
import mixserve.config as mconfig  # noqa: E402
import mixserve.engine as mengine  # noqa: E402
import mixserve.scheduler as msched  # noqa: E402

from paper_2503_11972_b200 import dropin  # noqa: E402

_base = dropin.SemanticCache
if __import__("os").environ.get("MC_DROPIN_FAKE"):  # host-logic check without a GPU (build container)
    from tests.fake_ring import FakeRing

    _base = type("FakeRingCache", (_base,), {"_ring_factory": staticmethod(FakeRing)})
dropin.install(mc, modules=(mconfig, mengine, msched), base=_base)

from mixserve.config import load_sim_config  # noqa: E402
from mixserve.engine import run_simulation  # noqa: E402
from mixserve.workload import generate_trace  # noqa: E402


def main():
    want = json.loads((ROOT / "tests" / "golden" / "sim_reports.json").read_text())
    out = {}
    for name, ref in sorted(want.items()):
        cfg = load_sim_config(ROOT / "baseline" / "_ref" / "configs" / f"{name}.cfg")
        trace = generate_trace(cfg.workload)
        result = run_simulation(cfg, trace)
        assert isinstance(result.cache, dropin.SemanticCache), type(result.cache)  # the GPU drop-in served it
        rep = json.loads(json.dumps(dataclasses.asdict(result.report), default=str))
        sha = hashlib.sha256(json.dumps(result.audit, sort_keys=True, default=str).encode()).hexdigest()
        out[name] = {"n_trace": len(trace), "report_equal": rep == ref["report"], "audit_equal": sha == ref["audit_sha"],
                     "hit_rate": rep.get("hit_rate"), "ref_hit_rate": ref["report"].get("hit_rate")}
        result.cache.close()
    print(json.dumps(out, sort_keys=True))


if __name__ == "__main__":
    main()
