"""Build librgb200.so (the sm_100a kernels + C ABI) in-tree with nvcc.

The shared library lands in paper_1604_01713_b200/_lib/librgb200.so so that it
travels with the repository snapshot to the GPU box.  nvcc cross-compiles for
sm_100a without a GPU.
"""

from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB_PATH = LIB_DIR / "librgb200.so"
SOURCES = ["rg_abi.cu", "rg_prof.cu", "rg_spmm.cu", "rg_tall.cu", "rg_qr.cu", "rg_steps.cu", "rg_cplx.cu", "rg_ilu.cu", "rg_halo.cu", "rg_dia.cu", "rg_peer.cu"]
HEADERS = ["rg_common.cuh"]
INCLUDE = PKG.parent / "include"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the rgb200 kernels need the CUDA 12.9 toolkit to build")


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    deps = [CSRC / s for s in SOURCES if (CSRC / s).exists()] + [CSRC / h for h in HEADERS]
    deps += list(INCLUDE.glob("*.h"))
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: pathlib.Path | None = None,
          extra_flags: list[str] | None = None) -> pathlib.Path:
    """Compile every .cu into librgb200.so (objects in parallel, then link).
    ``out`` / ``extra_flags`` build a variant library (A/B experiments)."""
    target = LIB_PATH if out is None else pathlib.Path(out)
    if out is None and not force and not _stale():
        return LIB_PATH
    LIB_DIR.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objdir = LIB_DIR / ("obj" if out is None else "obj_" + target.stem)
    objdir.mkdir(exist_ok=True)
    procs = []
    objs = []
    for src in SOURCES:
        path = CSRC / src
        if not path.exists():
            continue
        obj = objdir / (path.stem + ".o")
        objs.append(obj)
        # an object newer than its source and every header is current (each
        # objdir belongs to one flag set)
        hdrs = [CSRC / h for h in HEADERS] + list(INCLUDE.glob("*.h")) + [pathlib.Path(__file__)]
        if not force and obj.exists() and all(obj.stat().st_mtime > d.stat().st_mtime for d in [path, *hdrs]):
            continue
        cmd = [nvcc, *NVCC_FLAGS, *(extra_flags or []), "-c", str(path), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = []
    for src, pr in procs:
        out, _ = pr.communicate()
        if verbose and out:
            sys.stdout.write(out)
        if pr.returncode != 0:
            failed.append((src, out))
    if failed:
        msg = "\n".join(f"--- {s}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    target.parent.mkdir(parents=True, exist_ok=True)
    tmp = target.with_suffix(".so.tmp")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
                    *map(str, objs)], check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
