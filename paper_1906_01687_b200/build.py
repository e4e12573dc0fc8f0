"""In-tree build of the sm_100a engine (libgcpb.so) and the test oracles.

    python -m paper_1906_01687_b200.build          # engine + oracles
    python -m paper_1906_01687_b200.build --force  # rebuild everything

The engine is compiled with plain nvcc (-gencode arch=compute_100a,code=sm_100a
-lineinfo -O3), one object per .cu file in parallel, relinked when any object
changes.  The oracles are built by oracle/Makefile: liboracle.so (own C
restatement) always, oracle/_ref/libgcpref.so (the unmodified reference,
compiled in place) only when /root/reference is present.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / os.environ.get("GCPB_OBJDIR", "_build")
LIB = Path(os.environ.get("GCPB_LIB", PKG / "libgcpb.so"))
REFERENCE = Path("/root/reference/proj")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
]
SOURCES = ["gcpb.cu", "gcpb_fused_f32.cu", "gcpb_fused_f64.cu", "gcpb_io.cpp", "gcpb_host.cpp"]
_FUSED_DEPS = ["philox.cuh", "gcpb_kernels.cuh", "gcpb_fused.cuh"]
DEPS = {
    "gcpb.cu": ["philox.cuh", "gcpb_kernels.cuh", "gcpb_aux.cuh", "gcpb_gen.cuh",
                "gcpb_gen_host.inc", "rngstream.h", "gcpb_small.cuh"],
    "gcpb_fused_f32.cu": _FUSED_DEPS,
    "gcpb_fused_f64.cu": _FUSED_DEPS,
    "gcpb_io.cpp": [],
    "gcpb_host.cpp": [],
}


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def _compile(src: str, force: bool) -> tuple[str, bool]:
    s = CSRC / src
    o = OBJ / (Path(src).stem + ".o")
    deps = [s] + [CSRC / h for h in DEPS.get(src, [])]
    if src in ("gcpb.cu", "gcpb_io.cpp"):
        deps.append(ROOT / "include" / "gcpb.h")
    if not force and not _stale(o, deps):
        return src, False
    extra = os.environ.get("GCPB_NVFLAGS", "").split()
    cmd = [NVCC, *NVFLAGS, *extra, "-I", str(ROOT / "include"), "-c", str(s), "-o", str(o)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return src, True


def build_engine(force: bool = False, verbose: bool = True) -> Path:
    OBJ.mkdir(exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), SOURCES))
    objs = [OBJ / (Path(s).stem + ".o") for s in SOURCES]
    if force or any(changed for _, changed in results) or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lnccl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"[build] linked {LIB}")
    elif verbose:
        print(f"[build] {LIB} up to date")
    return LIB


def build_oracles(verbose: bool = True) -> None:
    targets = ["liboracle"]
    if REFERENCE.exists():
        # the reference itself, its acceptance gate, and the reference-side
        # binding of the engine (integration/gcp_b200.hpp) compiled against it
        targets += ["ref", "binding"]
    r = subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "-j8", *targets],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"[build] oracles: {', '.join(targets)}")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args(argv)
    build_engine(force=args.force)
    if not args.no_oracle:
        build_oracles()
    return 0


if __name__ == "__main__":
    sys.exit(main())
