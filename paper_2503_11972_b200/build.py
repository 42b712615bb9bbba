"""Build libmodmcache.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libmodmcache.so"
SOURCES = ["api.cu", "ring.cu", "scan_gemv.cu", "scan_stream8.cu", "scan_tc.cu", "rescore.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(exe).exists():
        raise RuntimeError("nvcc not found; cannot build libmodmcache.so")
    return exe


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "modmcache.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=()) -> Path:
    """Compile every source into libmodmcache.so (or `out`, with extra -D `defines`: A/B variants)."""
    lib = Path(out) if out else LIB
    if not out and not force and not needs_build():
        return LIB
    objdir = PKG / ("_build" if not out else "_build_" + lib.stem)
    objdir.mkdir(exist_ok=True)
    common = [
        "-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-O2", "-I", str(ROOT / "include"),
        "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3", *[f"-D{d}" for d in defines],
    ]
    jobs = []
    for src in SOURCES:  # one nvcc per translation unit, in parallel
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc(), *common, "-c", str(CSRC / src), "-o", str(obj)]
        jobs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    objs = []
    for src, obj, proc in jobs:
        out, err = proc.communicate()
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}\n{err}")
        if verbose:
            print(err, file=sys.stderr)
        objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_2503_11972_b200.build [--force] [-v] [--out PATH -DNAME=VALUE ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    print(build(force="--force" in args, verbose="-v" in args, out=out,
                defines=[a[2:] for a in args if a.startswith("-D")]))
