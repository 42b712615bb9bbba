"""gpurun_out/parity_gpu.jsonl (written by the GPU parity tests) -> profiles/parity_<tag>.txt.

North star: decisions bit-exact "with ties and near-threshold cases reported".  One row per
parity check: lookups, hits, exact ties, |s - tau| < 1e-12 (near_tau), runner-up within 1e-12
(near_tie), certificate fallbacks (exhaustive float64 rescan) and, for the golden op logs,
similarities bit-identical to the reference's own floats.

    python scripts/parity_report.py r02
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
rows = [json.loads(x) for x in (ROOT / "gpurun_out" / "parity_gpu.jsonl").read_text().splitlines() if x.strip()]
cols = ["queries", "hits", "exact_ties", "ties", "near_tau", "near_tie", "fallback", "ambiguous", "oracle_near_set",
        "sim_bit_equal"]
cols = [c for c in cols if any(c in r for r in rows)]
tot = {c: 0 for c in cols}
lines = [f"GPU parity checks ({len(rows)}), every one asserted against the oracle "
         "(decisions bit-exact; similarity within 1e-12, north-star tolerance 1e-3)", "",
         f"{'check':42s}" + "".join(f"{c:>16s}" for c in cols)]
for r in rows:
    lines.append(f"{r['check'][:42]:42s}" + "".join(f"{r.get(c, ''):>16}" for c in cols))
    for c in cols:
        tot[c] += int(r.get(c, 0) or 0)
lines += ["", f"{'TOTAL':42s}" + "".join(f"{tot[c]:>16}" for c in cols), "",
          "exact_ties/ties: two or more rows at the maximal float64 score (newest wins, flagged MC_FLAG_TIE)",
          "near_tau: best within 1e-12 of a threshold (MC_FLAG_NEAR_TAU); near_tie: runner-up within 1e-12 "
          "(MC_FLAG_NEAR_TIE)",
          "fallback: the certificate could not exclude an unscored row; the exhaustive float64 path answered",
          "ambiguous / oracle_near_set: the oracle's own argmax set within 1e-12 has > 1 row (numpy ulp "
          "instability, SURVEY.md §9 P5): the index is asserted to lie in that set"]
out = ROOT / "profiles" / f"parity_{tag}.txt"
out.write_text("\n".join(lines) + "\n")
print("\n".join(lines[-12:]))
