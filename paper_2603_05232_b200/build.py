"""Native build of the B200 library (sm_100a only).

Compiles paper_2603_05232_b200/csrc/*.cu with nvcc into the in-tree shared
library paper_2603_05232_b200/libslsp_b200.so (static cudart, so the .so has
no runtime-library search dependency). The library is the product; it is
loaded through the C ABI declared in include/slsp_b200.h.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libslsp_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["runtime.cu", "pack.cu", "lift.cu", "gemm.cu", "generic.cu"]
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared", "-cudart", "static",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
    f"-I{ROOT / 'include'}",
]


def _digest(src: str | None = None) -> str:
    """Content hash of the flags, the shared headers and `src` (all sources if None)."""
    import hashlib

    h = hashlib.sha256(" ".join(FLAGS).encode())
    srcs = SOURCES if src is None else [src]
    deps = sorted([CSRC / s for s in srcs] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")))
    deps.append(ROOT / "include" / "slsp_b200.h")
    for d in deps:
        h.update(d.name.encode())
        h.update(d.read_bytes())
    return h.hexdigest()


STAMP = PKG / "_build" / "stamp"


def _stale() -> bool:
    """Content-hash staleness (mtimes are unreliable across edits/snapshots)."""
    if not LIB.exists() or not STAMP.exists():
        return True
    return STAMP.read_text().strip() != _digest()


def _obj_stale(src: str) -> bool:
    obj = PKG / "_build" / (Path(src).stem + ".o")
    stamp = PKG / "_build" / (Path(src).stem + ".stamp")
    return not obj.exists() or not stamp.exists() or stamp.read_text().strip() != _digest(src)


def build_watchdog() -> Path:
    """Debug variant libslsp_b200_wd.so (-DSLSP_WATCHDOG: stuck mbarrier waits
    print and trap); load it with SLSP_LIB=<path>. Never used by the product."""
    out = PKG / "libslsp_b200_wd.so"
    srcs = [str(CSRC / s) for s in SOURCES]
    cmd = [NVCC, *[f for f in FLAGS if f not in ("-cudart", "static")], "-cudart", "static", "-DSLSP_WATCHDOG",
           *srcs, "-o", str(out)]
    subprocess.run(cmd, check=True)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    objs = []
    build_dir = PKG / "_build"
    build_dir.mkdir(exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = build_dir / (Path(src).stem + ".o")
        objs.append(str(obj))
        if not force and not _obj_stale(src):  # per-object content hash: rebuild only what changed
            continue
        cmd = [NVCC, *[f for f in FLAGS if f not in ("-shared",)], "-c", str(CSRC / src), "-o", str(obj)]
        cmd = [c for c in cmd if c not in ("-cudart", "static")]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(f"[nvcc {src}]\n{out}")
        failed |= p.returncode != 0
        if p.returncode == 0:
            (build_dir / (Path(src).stem + ".stamp")).write_text(_digest(src))
    if failed:
        raise RuntimeError("nvcc failed")
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
            "-Xcompiler", "-fPIC", *objs, "-o", str(LIB)]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    STAMP.write_text(_digest())
    return LIB


if __name__ == "__main__":
    if "--watchdog" in sys.argv:
        print(build_watchdog())
        sys.exit(0)
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
