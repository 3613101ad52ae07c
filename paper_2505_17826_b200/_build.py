"""Build libtg_loss.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2505_17826_b200._build [--verbose]

Outputs ``paper_2505_17826_b200/_lib/libtg_loss.so``.  The CUDA runtime is
linked statically, so the library only needs the driver at load time.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libtg_loss.so"
OBJDIR = ROOT / "build" / "obj"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-I", str(ROOT / "include"), "-I", str(CSRC)]
CU_SOURCES = ["tg_fused_tma.cu", "tg_stream.cu", "tg_group.cu", "tg_pack.cu", "tg_lmhead.cu",
              "tg_gemm.cu", "tg_update.cu", "tg_adamw.cu", "tg_api.cu"]
CPP_SOURCES = ["tg_host.cpp"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (res.stdout or res.stderr):
        sys.stderr.write(res.stdout + res.stderr)
    return res


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


# builds for kernel studies (never the product library):
#   prof -> libtg_loss_prof.so with per-CTA cycle accounting in k_fused_tma
#   ab   -> libtg_loss_ab.so: the run-time A/B switches (TG_FUSED_CL, TG_FUSED_IMPL=2
#           with the L2-reread kernel tg_fused_l2.cu, TG_FWD_TMA, TG_PREFETCH_ROWS,
#           TG_FUSED_ANCHOR, TG_LMHEAD_PAIR / _ORDER); tests/test_gpu_alt_paths.py
VARIANTS = {"prof": ["-DTG_FUSED_PROF"], "ab": ["-DTG_AB_SWITCHES"]}
EXTRA_SOURCES = {"ab": ["tg_fused_l2.cu"]}
AB_LIB = LIBDIR / "libtg_loss_ab.so"


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False,
          variant: str | None = None, defines: list | None = None) -> Path:
    objdir, lib_out = OBJDIR, LIB
    defines = list(defines or [])
    if variant:
        objdir = ROOT / "build" / f"obj_{variant}"
        lib_out = LIBDIR / f"libtg_loss_{variant}.so"
        defines = VARIANTS.get(variant, []) + defines
    OBJDIR_, LIB_ = objdir, lib_out
    OBJDIR_.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "tg_loss.h"]
    objs = []
    extra_src = EXTRA_SOURCES["ab"] if "-DTG_AB_SWITCHES" in defines else []
    for src in CU_SOURCES + extra_src:
        obj = OBJDIR_ / (src + ".o")
        objs.append(obj)
        if force or _stale(obj, [CSRC / src, *headers]):
            extra = ["-Xptxas", "-v"] if ptxas_verbose else []
            _run([nvcc(), *ARCH, *NVCC_FLAGS, *defines, *extra, "-c", str(CSRC / src), "-o",
                  str(obj)],
                 verbose or ptxas_verbose)
    for src in CPP_SOURCES:
        obj = OBJDIR_ / (src + ".o")
        objs.append(obj)
        if force or _stale(obj, [CSRC / src, *headers]):
            _run(["g++", "-O2", "-std=c++17", "-fPIC", "-I", str(ROOT / "include"), "-c",
                  str(CSRC / src), "-o", str(obj)], verbose)
    if force or _stale(LIB_, objs):
        # --no-undefined: a missing definition fails the build, not the dlopen
        _run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-Xlinker", "--no-undefined",
              "-o", str(LIB_), *map(str, objs)], verbose)
    return LIB_


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), None)
    defs = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--define=")]
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv,
                ptxas_verbose="--ptxas" in sys.argv, variant=var, defines=defs))
