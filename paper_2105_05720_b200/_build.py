"""In-tree builders for the native parts of the package.

libcoconet_cuda.so   : csrc/*.cu, sm_100a only (-gencode arch=compute_100a,code=sm_100a),
                       static cudart, no torch dependency (pure C-ABI).
libcoconet_engine.so : csrc/engine/*.cpp — GpuEngine, the drop-in host that
                       walks a ccopt Program; compiled against the reference's
                       own DSL headers (the drop-in surface), so it is only
                       (re)built where those headers exist.
oracle/_build, oracle/_ref : the parity checker (oracle/Makefile).
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CCOPT_REF_DIR = Path(os.environ.get("CCOPT_REF_DIR", "/root/reference/proj"))
NLOHMANN_DIR = Path(
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")

CUDA_LIB = PKG / "libcoconet_cuda.so"
ENGINE_LIB = PKG / "libcoconet_engine.so"

CU_SOURCES = ["context.cu", "tlist.cu", "fused_opt.cu", "gen.cu", "collectives.cu",
              "fused_bdr.cu", "gemm_tc.cu", "pointwise.cu", "unfused.cu", "heap_cumem.cu"]


def _run(cmd, cwd=None):
    proc = subprocess.run(cmd, cwd=cwd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"command failed ({proc.returncode}): {' '.join(map(str, cmd))}\n{proc.stdout}")
    return proc.stdout


def _stale(target: Path, sources) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(s).stat().st_mtime > t for s in sources)


def build_cuda(force: bool = False, verbose: bool = False, jobs: int = 8) -> Path:
    srcs = [CSRC / s for s in CU_SOURCES if (CSRC / s).exists()]
    deps = srcs + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [INCLUDE / "coconet_cuda.h"]
    if not force and not _stale(CUDA_LIB, deps):
        return CUDA_LIB
    objdir = PKG / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(INCLUDE),
                    "-I", str(CSRC), "--expt-relaxed-constexpr", "-Xptxas", "-v"]
    procs = []
    objs = []
    for s in srcs:
        o = objdir / (s.stem + ".o")
        objs.append(o)
        cmd = [NVCC, "-c", str(s), "-o", str(o)] + flags
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
    logs = []
    for cmd, p in procs:
        out, _ = p.communicate()
        logs.append(out)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{out}")
    (PKG / "build" / "ptxas.log").write_text("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    _run([NVCC, "-shared", "-o", str(CUDA_LIB)] + [str(o) for o in objs] + ARCH +
         ["-cudart", "static", "-lcuda"])
    return CUDA_LIB


def build_engine(force: bool = False) -> Path | None:
    srcs = sorted((CSRC / "engine").glob("*.cpp")) if (CSRC / "engine").exists() else []
    if not srcs:
        return None
    hdrs = list((INCLUDE / "coconet").glob("*.hpp")) + [INCLUDE / "coconet_cuda.h"]
    if not (CCOPT_REF_DIR / "include" / "ccopt").exists():
        # The DSL headers are the reference's; without them keep the prebuilt
        # library (it travels with the tree).
        return ENGINE_LIB if ENGINE_LIB.exists() else None
    if not force and not _stale(ENGINE_LIB, srcs + hdrs):
        return ENGINE_LIB
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-pthread", "-I", str(INCLUDE),
           "-I", str(CCOPT_REF_DIR / "include"), "-I", str(NLOHMANN_DIR), "-I",
           str(CUDA_HOME / "include"), "-o", str(ENGINE_LIB)] + [str(s) for s in srcs] + [
        "-L", str(PKG), "-Wl,-rpath,$ORIGIN", "-lcoconet_cuda",
        "-L", str(CUDA_HOME / "lib64"), "-Wl,-rpath," + str(CUDA_HOME / "lib64"), "-lcudart"]
    _run(cmd)
    return ENGINE_LIB


CLI_BIN = PKG / "coconet-ccopt"


def build_cli(force: bool = False) -> Path | None:
    """coconet-ccopt: the reference CLI flow (tools/ccopt.cpp) with a CUDA
    backend; like the engine it needs the reference DSL headers to build."""
    srcs = sorted((CSRC / "cli").glob("*.cpp")) if (CSRC / "cli").exists() else []
    if not srcs:
        return None
    hdrs = list((INCLUDE / "coconet").glob("*.hpp")) + [INCLUDE / "coconet_cuda.h"]
    if not (CCOPT_REF_DIR / "include" / "ccopt").exists():
        return CLI_BIN if CLI_BIN.exists() else None
    if not force and not _stale(CLI_BIN, srcs + hdrs):
        return CLI_BIN
    cmd = ["g++", "-std=c++20", "-O2", "-pthread", "-I", str(INCLUDE),
           "-I", str(CCOPT_REF_DIR / "include"), "-I", str(NLOHMANN_DIR), "-I",
           str(CUDA_HOME / "include"), "-o", str(CLI_BIN)] + [str(s) for s in srcs] + [
        "-L", str(PKG), "-Wl,-rpath,$ORIGIN", "-lcoconet_cuda",
        "-L", str(CUDA_HOME / "lib64"), "-Wl,-rpath," + str(CUDA_HOME / "lib64"), "-lcudart"]
    _run(cmd)
    return CLI_BIN


def build_oracle() -> None:
    make = shutil.which("make")
    if not make:
        return
    targets = ["c"]
    if (CCOPT_REF_DIR / "include" / "ccopt").exists():
        targets.append("ref")
    _run([make, "-s", "-C", str(ROOT / "oracle")] + targets)


def build_all(force: bool = False) -> None:
    build_cuda(force=force)
    build_engine(force=force)
    build_cli(force=force)
    build_oracle()
