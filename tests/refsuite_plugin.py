"""pytest plugin: run the REFERENCE's own test suite against the GPU drop-in.

Loaded with ``-p tests.refsuite_plugin`` on ``baseline/_ref/tests`` (staged by
scripts/stage_reference.sh).  Before any test module imports ``mixserve``, it
installs the drop-in into ``mixserve.cache`` (paper_2503_11972_b200.dropin),
so ``SimConfig.build_cache()`` (config.py:98-104), ``scheduler.classify``,
``Simulation`` and the tests themselves all run on the device ring.
MC_DROPIN_FAKE=1 swaps the device ring for the CPU FakeRing (host-logic check
in the build container, which has no GPU).
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "baseline" / "_ref")):
    if p not in sys.path:
        sys.path.insert(0, p)

import mixserve.cache as _mc  # noqa: E402

from paper_2503_11972_b200 import SemanticCache, dropin  # noqa: E402

_base = SemanticCache
if os.environ.get("MC_DROPIN_FAKE"):
    from tests.fake_ring import FakeRing

    _base = type("FakeRingCache", (SemanticCache,), {"_ring_factory": staticmethod(FakeRing)})
dropin.install(_mc, base=_base)


def pytest_report_header(config):
    return f"mixserve.cache.SemanticCache -> {_mc.SemanticCache.__mro__[1].__module__}.{_mc.SemanticCache.__mro__[1].__name__}"
