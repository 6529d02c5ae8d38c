"""Build liblapb200.so (the sm_100a CUDA library behind the C ABI).

Compiles every csrc/*.cu with nvcc for sm_100a into an in-tree shared
library (paper_1311_1695_b200/_lib/liblapb200.so).  cudart is linked
statically so the library does not depend on the CUDA runtime torch ships.
Host code is compiled with -ffp-contract=off so the IC(0) factorization stays
bit-exact with the reference's (ic0.py:48-78).

Usage:  python -m paper_1311_1695_b200.build  [--force] [--jobs N]
"""

import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIBDIR = HERE / "_lib"
LIB = LIBDIR / "liblapb200.so"
OBJDIR = HERE.parent / "build" / "obj"
INCLUDE = HERE.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-ffp-contract=off", "-Xcompiler", "-fopenmp", "-Xptxas", "-v",
    f"-I{INCLUDE}",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def up_to_date():
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def _compile(src):
    obj = OBJDIR / (src.stem + ".o")
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
    (OBJDIR / (src.stem + ".ptxas.txt")).write_text(res.stderr)
    return obj


def build(force=False, jobs=None, verbose=False):
    """Compile and link the library; returns its path."""
    if not force and up_to_date():
        return LIB
    OBJDIR.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    srcs = sources()
    with ThreadPoolExecutor(max_workers=jobs or min(8, len(srcs))) as ex:
        objs = list(ex.map(_compile, srcs))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", *map(str, objs),
           "-o", str(tmp), "-lgomp", "-lpthread", "-ldl", "-lrt"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_variant(name, defines):
    """An alternative build with extra -D flags into build/variants/<name>.so
    (A/B experiments: run with LG_LIB_OVERRIDE=build/variants/<name>.so)."""
    vdir = HERE.parent / "build" / "variants"
    odir = vdir / (name + "_obj")
    odir.mkdir(parents=True, exist_ok=True)
    flags = [f"-D{d}" for d in defines]

    def comp(src):
        obj = odir / (src.stem + ".o")
        res = subprocess.run([nvcc(), *ARCH, *NVCC_FLAGS, *flags, "-c", str(src), "-o", str(obj)],
                             capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
        (odir / (src.stem + ".ptxas.txt")).write_text(res.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=8) as ex:
        objs = list(ex.map(comp, sources()))
    out = vdir / (name + ".so")
    res = subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", *map(str, objs),
                          "-o", str(out), "-lgomp", "-lpthread", "-ldl", "-lrt"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--variant", nargs="+", metavar=("NAME", "DEFINE"),
                    help="build build/variants/NAME.so with -DDEFINE ... instead")
    args = ap.parse_args(argv)
    if args.variant:
        print(build_variant(args.variant[0], args.variant[1:]))
        return 0
    build(force=args.force, jobs=args.jobs, verbose=True)


if __name__ == "__main__":
    sys.exit(main())
