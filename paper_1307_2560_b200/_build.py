"""Build recipe for the native libraries (nvcc / g++ invoked directly, in-tree).

  libychg_b200.so  CUDA kernels for sm_100a + the C ABI (include/ychg_b200.h)
  libychg.so       the C++ drop-in (namespace ychg, include/ychg/*.hpp) over the C ABI

Both land next to this file so they travel to the GPU box with the repo
snapshot.  Re-running is incremental on source mtimes.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")

CUDA_SO = os.path.join(PKG, "libychg_b200.so")
CXX_SO = os.path.join(PKG, "libychg.so")
CLI_BIN = os.path.join(PKG, "ychg_b200")

NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SRCS = ["ychg_scan.cu", "ychg_aux.cu", "ychg_profile.cu", "ychg_decompose.cu", "ychg_capi.cu"]
CU_DEPS = CU_SRCS + ["ychg_device.cuh", "ychg_kernels.h"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the yCHG kernels need the CUDA 12.9 toolkit")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose_ptxas: bool = False, force: bool = False) -> None:
    deps = [os.path.join(CSRC, f) for f in CU_DEPS] + [os.path.join(INCLUDE, "ychg_b200.h")]
    if force or _stale(CUDA_SO, deps):
        cmd = [_nvcc(), *NVCC_ARCH, "-lineinfo", "-O3", "-std=c++17", "--shared",
               "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I" + INCLUDE,
               "-o", CUDA_SO, *[os.path.join(CSRC, f) for f in CU_SRCS]]
        if verbose_ptxas:
            cmd.insert(1, "-Xptxas=-v")
        _run(cmd)
    cxx_deps = [os.path.join(CSRC, "ychg_runscan.cpp"), CUDA_SO] + [
        os.path.join(INCLUDE, "ychg", f) for f in ("errors.hpp", "image.hpp", "runscan.hpp", "scan_b200.hpp", "pnm.hpp")]
    if force or _stale(CXX_SO, cxx_deps):
        _run([os.environ.get("CXX", "g++"), "-std=c++20", "-O2", "-fPIC", "-shared", "-I" + INCLUDE,
              "-o", CXX_SO, os.path.join(CSRC, "ychg_runscan.cpp"), "-L" + PKG, "-l:libychg_b200.so",
              "-Wl,-rpath,$ORIGIN"])
    cli_deps = [os.path.join(CSRC, "ychg_cli.cpp"), CXX_SO, CUDA_SO]
    if force or _stale(CLI_BIN, cli_deps):
        _run([os.environ.get("CXX", "g++"), "-std=c++20", "-O2", "-I" + INCLUDE, "-o", CLI_BIN,
              os.path.join(CSRC, "ychg_cli.cpp"), "-L" + PKG, "-l:libychg.so", "-l:libychg_b200.so",
              "-Wl,-rpath,$ORIGIN"])


def build_variant(warps: int, stages: int, *defines: str) -> str:
    """Experimental launch-shape / diagnostics variants (benchmarking only):
    libychg_b200_w{W}s{S}[_define...].so."""
    tag = "".join("_" + d.lower().replace("ychg_", "") for d in defines)
    out = os.path.join(PKG, f"libychg_b200_w{warps}s{stages}{tag}.so")
    _run([_nvcc(), *NVCC_ARCH, "-lineinfo", "-O3", "-std=c++17", "--shared", f"-DYCHG_WARPS={warps}",
          f"-DYCHG_STAGES={stages}", *[f"-D{d}" for d in defines], "-Xcompiler", "-fPIC,-fvisibility=hidden",
          "-I" + INCLUDE, "-o", out, *[os.path.join(CSRC, f) for f in CU_SRCS]])
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        build_variant(int(sys.argv[i + 1]), int(sys.argv[i + 2]), *sys.argv[i + 3:])
    else:
        build(verbose_ptxas="-v" in sys.argv, force="-f" in sys.argv)
