"""Build libspecdec_b200.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "lib")
LIB = os.path.join(OUT, "libspecdec_b200.so")
PROBE_LIB = os.path.join(OUT, "probe", "libspecdec_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr"]
SOURCES = ["model.cu", "check_kernels.cu", "step_kernels.cu", "fast_kernels.cu", "gemm_sm100.cu", "gemm_cluster.cu", "capi.cpp",
           "engine.cpp", "session.cpp", "comm.cpp"]


def _obj(src: str) -> str:
    return os.path.join(OUT, "obj", src + ".o")


def _needs(src: str) -> bool:
    o = _obj(src)
    if not os.path.exists(o):
        return True
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(PKG, "..", "include", "specdec_b200.h"))
    t = os.path.getmtime(o)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str) -> None:
    os.makedirs(os.path.join(OUT, "obj"), exist_ok=True)
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", _obj(src)]
    if src.endswith(".cpp"):
        cmd.insert(1, "-x")
        cmd.insert(2, "cu")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)


def build(verbose: bool = False) -> str:
    todo = [s for s in SOURCES if _needs(s)]
    with ThreadPoolExecutor(max_workers=min(8, len(todo) or 1)) as ex:
        list(ex.map(_compile, todo))
    if todo or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *[_obj(s) for s in SOURCES]]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    if verbose:
        print("built", LIB)
    return LIB


def build_probe() -> str:
    """A measurement-only variant of the library whose GEMM honours the
    bottleneck probes of sd_debug_gemm (-DSD_GEMM_PROBE); tools/ load it with
    --lib.  The library itself never contains them."""
    build()
    os.makedirs(os.path.dirname(PROBE_LIB), exist_ok=True)
    po = os.path.join(OUT, "probe", "gemm_sm100.cu.o")
    cmd = [NVCC, *ARCH, *FLAGS, "-DSD_GEMM_PROBE", "-c", os.path.join(CSRC, "gemm_sm100.cu"), "-o", po]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    objs = [po if s == "gemm_sm100.cu" else _obj(s) for s in SOURCES]
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", PROBE_LIB, *objs], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return PROBE_LIB


if __name__ == "__main__":
    if "--probe" in sys.argv:
        print("built", build_probe())
    else:
        build(verbose=True)
