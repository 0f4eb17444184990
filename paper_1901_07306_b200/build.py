"""Build libsspd_b200.so in-tree with nvcc for sm_100a.

The library is the C-ABI product (include/sspd_b200.h); Python loads it
with ctypes (see _lib.py).  It is built in-tree so the same .so travels to
the GPU box with the repository snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB_PATH = LIB_DIR / "libsspd_b200.so"
SOURCES = ["scan.cu", "scan_smem.cu", "scan_bpart.cu", "estimate.cu", "sliding.cu", "merge.cu", "ingest.cu", "exact.cu", "abi.cu", "host_stage.cu", "radix.cu"]
HEADERS = ["sspd_common.cuh", "launch.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "sspd_b200.h"]
    return any(d.stat().st_mtime > built for d in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None) -> Path:
    """Compile every CUDA source into one shared library (idempotent).  `out`
    (tuning A/B builds only) writes the library elsewhere."""
    if out is None and not force and not _stale():
        return LIB_PATH
    lib_path = Path(out) if out is not None else LIB_PATH
    LIB_DIR.mkdir(exist_ok=True)
    objs = []
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                    "-I", str(ROOT / "include"), "-Xptxas", "-v" if verbose else "-O3"]
    flags += os.environ.get("SSPD_NVCC_FLAGS", "").split()  # A/B builds of compile-time knobs
    for src in SOURCES:
        obj = LIB_DIR / (Path(src).stem + f".{os.getpid()}.o")
        cmd = [NVCC, "-c", str(CSRC / src), "-o", str(obj)] + flags
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
        if verbose and res.stderr:
            print(res.stderr, file=sys.stderr)
        objs.append(str(obj))
    tmp = lib_path.with_suffix(".so.tmp")
    cmd = [NVCC, "-shared", "-o", str(tmp)] + ARCH + [*objs, "-cudart", "static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, lib_path)
    for o in objs:
        os.unlink(o)
    return lib_path


def build_hostfast(force: bool = False) -> Path:
    """The CPython binding of the drop-in staging copy (csrc/hostfast.c),
    compiled with the host C compiler next to the package (host code only;
    Python falls back to the ctypes call when it is absent)."""
    import sysconfig

    src = CSRC / "hostfast.c"
    out = PKG / ("_hostfast" + sysconfig.get_config_var("EXT_SUFFIX"))
    if not force and out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    cc = os.environ.get("CC", "gcc")
    tmp = out.with_suffix(".tmp")
    cmd = [cc, "-O2", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"], str(src), "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"{cc} failed for hostfast.c:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    outs = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=Path(outs[0]) if outs else None))
    if not outs:
        print(build_hostfast(force="--force" in sys.argv))
