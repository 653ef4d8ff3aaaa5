"""Build the B200 engine in-tree (no JIT cache), so it travels with the repo
snapshot to the GPU box:

* libb2conv.so       — every kernel and the C ABI (include/b2conv.h), nvcc for
                       sm_100a, no torch headers;
* _b2conv_torch.so   — the PyTorch operator library (torch.ops.b2conv.*,
                       csrc/torch_ext.cpp), g++ against torch's headers, linked
                       to libb2conv.so through $ORIGIN.

    python -m paper_2103_16234_b200.build [--force]

B2C_DEV_BUILD=1 adds -DB2C_DEV (development instrumentation: role skipping,
per-CTA traces, cycle dumps); release builds compile it out.
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
LIB = PKG / "libb2conv.so"
TORCH_LIB = PKG / "_b2conv_torch.so"
TORCH_SRC = CSRC / "torch_ext.cpp"
SOURCES = [CSRC / "conv_launch.cu", CSRC / "conv_tc.cu", CSRC / "probe.cu", CSRC / "api.cpp"]
DEPS = SOURCES + [CSRC / "conv_kernel.cuh", CSRC / "conv1x1_vec.cuh", CSRC / "conv_tc.cuh", CSRC / "conv_row.cuh",
                  CSRC / "conv1x1_ws.cuh", CSRC / "conv1x1_tma.cuh", CSRC / "ptx.cuh", CSRC / "internal.h", ROOT / "include" / "b2conv.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# No --use_fast_math / -ftz: denormals and IEEE rounding must match numpy.
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
if os.environ.get("B2C_DEV_BUILD"):
    NVFLAGS.append("-DB2C_DEV")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 engine has no CPU fallback and must be compiled")


def stale() -> bool:
    if not LIB.exists() or not TORCH_LIB.exists():
        return True
    t = min(LIB.stat().st_mtime, TORCH_LIB.stat().st_mtime)
    return any(p.stat().st_mtime > t for p in DEPS + [TORCH_SRC])


def build_torch_ext() -> Path:
    """The operator library: a thin torch adapter over the C ABI."""
    import torch
    from torch.utils import cpp_extension as ce

    tdir = Path(torch.__file__).resolve().parent
    abi = "1" if torch.compiled_with_cxx11_abi() else "0"
    cxx = shutil.which("g++") or "g++"
    tmp = TORCH_LIB.with_suffix(".so.tmp")
    cuda_inc = str(Path(ce.CUDA_HOME or "/usr/local/cuda") / "include")
    cmd = [cxx, "-O2", "-std=c++17", "-fPIC", "-shared", f"-D_GLIBCXX_USE_CXX11_ABI={abi}",
           "-I", str(tdir / "include"), "-I", str(tdir / "include" / "torch" / "csrc" / "api" / "include"),
           "-I", cuda_inc, "-I", str(ROOT / "include"), str(TORCH_SRC), "-o", str(tmp),
           "-L", str(tdir / "lib"), "-lc10", "-lc10_cuda", "-ltorch_cpu",
           "-L", str(PKG), "-l:libb2conv.so", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build of _b2conv_torch.so failed")
    os.replace(tmp, TORCH_LIB)
    return TORCH_LIB


def build_dev_variant() -> Path:
    """libb2conv_dev.so: the same sources with -DB2C_DEV (development switches
    and instrumentation), loaded by _native when B2C_LIB_VARIANT=dev — for
    A/B runs on the GPU box only; never the product library."""
    objdir = PKG / "build_dev"
    objdir.mkdir(exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = objdir / (src.stem + ".o")
        return obj, subprocess.run([nvcc(), *ARCH, *NVFLAGS, "-DB2C_DEV", "-c", str(src), "-o", str(obj)],
                                   capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stderr)
            raise RuntimeError("nvcc failed (dev variant)")
    out = PKG / "libb2conv_dev.so"
    r = subprocess.run([nvcc(), *ARCH, "-shared", "-Xlinker", "-soname=libb2conv_dev.so", "-o", str(out),
                        *[str(o) for o, _ in results], "-lcudart_static", "-lpthread", "-ldl", "-lrt"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stderr)
        raise RuntimeError("link of libb2conv_dev.so failed")
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc(), *ARCH, *NVFLAGS, "-c", str(src), "-o", str(obj)]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs, log = [], []
    for src, obj, r in results:
        log.append(r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src.name}")
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-Xlinker", "-soname=libb2conv.so", "-o", str(tmp), *objs, "-lcudart_static",
           "-lpthread", "-ldl", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libb2conv.so failed")
    os.replace(tmp, LIB)
    (objdir / "ptxas.log").write_text("".join(log))
    build_torch_ext()
    if verbose:
        print("".join(log))
    return LIB


if __name__ == "__main__":
    if "--dev" in sys.argv:
        print(build_dev_variant())
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
