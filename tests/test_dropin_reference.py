"""Drop-in proof under the reference's own control plane.

1. The reference's complete test suite (pkg/tests, 193 tests) runs with
   ``mixserve.cache.SemanticCache`` replaced by the GPU drop-in
   (tests/refsuite_plugin.py -> paper_2503_11972_b200.dropin.install).
2. The reference Simulation on its four shipped configs, with the drop-in
   installed, reproduces the report and the per-request audit of the stock run
   (recorded by tests/golden/make_sim_golden.py).
Both need the staged reference (scripts/stage_reference.sh -> baseline/_ref);
the self-contained counterpart — the same Simulations' cache traffic replayed
from committed op logs (tests/golden/sim_*.npz) — runs in
tests/test_gpu_parity.py::test_golden_op_logs.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "tests").is_dir() or not (REF / "mixserve").is_dir(),
                                 reason="reference not staged (scripts/stage_reference.sh)")]


def _run(cmd, timeout):
    env = dict(os.environ)
    env.pop("MC_DROPIN_FAKE", None)
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_reference_suite_passes_with_the_gpu_cache():
    r = _run([sys.executable, "-m", "pytest", "-p", "tests.refsuite_plugin", str(REF / "tests"), "-q",
              "-p", "no:cacheprovider"], timeout=1500)
    tail = "\n".join(r.stdout.strip().splitlines()[-15:])
    print(tail)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "reference_suite_on_gpu.txt").write_text(r.stdout[-20000:] + r.stderr[-5000:])
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail


def test_reference_simulations_identical_with_the_gpu_cache():
    r = _run([sys.executable, str(ROOT / "tests" / "dropin_sim.py")], timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    print(json.dumps(res, indent=1))
    assert len(res) == 4
    for name, v in res.items():
        assert v["report_equal"] and v["audit_equal"], (name, v)
