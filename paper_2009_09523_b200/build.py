"""In-tree build of every native artefact (sm_100a only).

  libvnt_engine.so  CUDA engine + C-ABI (include/vnt_engine.h)
  libvnt.so         C++ drop-in `vnt::` API (include/vnt/*.hpp) + its C-ABI
                    (include/vnt_trainer.h), linked against the engine
  build/tests/*     C++ drop-in tests (tests/cpp/*.cpp)
  oracle/_build, oracle/_ref   test-only CPU oracles (oracle/Makefile)
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
INC = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_LIB = "/usr/local/cuda/lib64"
# Link the NCCL that torch ships (2.28.x): one libnccl.so.2 per process, so
# torch.distributed and the engine can share a process in either load order.
try:
    import nvidia.nccl as _nccl
    NCCL_ROOT = Path(list(_nccl.__path__)[0])
except Exception:  # pragma: no cover
    NCCL_ROOT = None


def _run(cmd, cwd=ROOT):
    print("+", " ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True, cwd=cwd)


def _stale(out: Path, deps) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def nccl_flags():
    if NCCL_ROOT and (NCCL_ROOT / "lib" / "libnccl.so.2").exists():
        lib = NCCL_ROOT / "lib"
        return [f"-I{NCCL_ROOT / 'include'}", f"-L{lib}", "-l:libnccl.so.2",
                "-Xlinker", f"-rpath={lib}"]
    return ["-lnccl"]


def build_engine(force=False) -> Path:
    out = PKG / "libvnt_engine.so"
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [INC / "vnt_engine.h"]
    if force or _stale(out, deps):
        _run([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v" if os.environ.get("VNT_PTXAS_VERBOSE") else "-O3",
              "-shared", "-o", out, CSRC / "engine.cu", *nccl_flags(), "-lcuda"])
    return out


def build_host(force=False) -> Path | None:
    out = PKG / "libvnt.so"
    srcs = sorted(HOST.glob("*.cpp"))
    if not srcs:
        return None
    deps = srcs + list(INC.glob("vnt/*.hpp")) + [INC / "vnt_trainer.h", PKG / "libvnt_engine.so"]
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-shared", f"-I{INC}",
              f"-I/usr/local/cuda/include", "-o", out, *srcs,
              f"-L{PKG}", "-lvnt_engine", f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,$ORIGIN",
              "-lpthread"])
    return out


def build_cpp_tests(force=False):
    tdir = ROOT / "tests" / "cpp"
    bdir = ROOT / "build" / "tests"
    bdir.mkdir(parents=True, exist_ok=True)
    outs = []
    for src in sorted(tdir.glob("test_*.cpp")):
        out = bdir / src.stem
        if force or _stale(out, [src, PKG / "libvnt.so", tdir / "check.hpp"]):
            _run(["g++", "-std=c++20", "-O2", f"-I{INC}", f"-I{tdir}", "-o", out, src,
                  f"-L{PKG}", "-lvnt", "-lvnt_engine", f"-Wl,-rpath,{PKG}", "-lpthread"])
        outs.append(out)
    return outs


NLOHMANN = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty")


def build_tools(force=False):
    """`vnt_train` — the reference CLI's train command over the drop-in Trainer."""
    src = PKG / "tools" / "vnt_train.cpp"
    out = ROOT / "build" / "bin" / "vnt_train"
    out.parent.mkdir(parents=True, exist_ok=True)
    if not (NLOHMANN / "nlohmann" / "json.hpp").exists():
        print("nlohmann/json.hpp not found; skipping vnt_train")
        return None
    if force or _stale(out, [src, PKG / "libvnt.so"]):
        _run(["g++", "-std=c++20", "-O2", f"-I{INC}", f"-I{NLOHMANN}", "-o", out, src,
              f"-L{PKG}", "-lvnt", "-lvnt_engine", f"-Wl,-rpath,{PKG}", "-lpthread"])
    return out


def build_oracle():
    """Test-only: our C restatement always; the reference itself when present."""
    _run(["make", "-s", "-C", ROOT / "oracle", "oracle"])
    if Path("/root/reference/proj/core/src").exists():
        _run(["make", "-s", "-j8", "-C", ROOT / "oracle", "ref"])


def build_all(force=False):
    build_engine(force)
    if build_host(force):
        build_cpp_tests(force)
        build_tools(force)
    build_oracle()


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv)
