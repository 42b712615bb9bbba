"""Opcode evidence from the built library (cuobjdump -sass): per kernel, the Blackwell-native
instructions that prove the tcgen05 / TMA / TMEM paths, plus the dp4a and float64 counts.

    python scripts/sass_summary.py r02   ->  profiles/sass_r02.txt
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
lib = ROOT / "paper_2503_11972_b200" / "libmodmcache.so"
sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
WANT = ["UTCHMMA", "UTCIMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "UTMALDG", "UBLKCP", "SYNCS", "IDP.4A", "DFMA", "DADD",
        "DMUL", "ATOMG.E.CAS", "REDG", "LDG", "STG", "ST.E"]
per = collections.defaultdict(collections.Counter)
sizes = collections.Counter()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if cur and m:
        op = m.group(1)
        sizes[cur] += 1
        for w in WANT:
            if op.startswith(w):
                per[cur][op] += 1


def short(name):
    m = re.search(r"_ZN2mc\d+(\w+?)(I|E)", name)
    base = m.group(1) if m else name[:40]
    t = re.search(r"ILi(\d+)ELi(\d+)E(?:Lb(\d)E|Li(\d+)E)", name)
    return base + (f"<{','.join(x for x in t.groups() if x is not None)}>" if t else "")


lines = [f"cuobjdump -sass {lib.name} ({len(sizes)} kernels); counts of selected opcodes per kernel", ""]
for k in sorted(per, key=lambda k: short(k)):
    if not any(o.startswith(("UTC", "LDTM", "UTMA", "UBLK", "IDP", "D")) for o in per[k]):
        continue
    ops = ", ".join(f"{o} {n}" for o, n in sorted(per[k].items()))
    lines.append(f"{short(k):34s} {sizes[k]:6d} instr | {ops}")
(ROOT / "profiles" / f"sass_{tag}.txt").write_text("\n".join(lines) + "\n")
print("\n".join(lines))
