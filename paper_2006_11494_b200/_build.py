"""In-tree build of the B200 library and its Python binding.

* ``lib/libtrilist_b200.so`` -- the CUDA kernels + the C-ABI of
  ``include/trilist_b200.h`` (nvcc, ``-gencode arch=compute_100a,code=sm_100a``,
  cudart linked statically so the .so is self-contained on the GPU box).
* ``trilist/_core*.so`` -- the pybind11 mirror of the reference's
  ``trilist._core`` over the C++ facade (``include/trilist_b200/trilist.hpp``).

Incremental: a target is rebuilt only when a source it depends on is newer.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libtrilist_b200.so")
EXT = os.path.join(PKG, "trilist", "_core" + sysconfig.get_config_var("EXT_SUFFIX"))
CLI = os.path.join(PKG, "bin", "trilist")

CU_SOURCES = ["tl_build.cu", "tl_aot.cu", "tl_parse.cu", "tl_orders.cu", "tl_verify.cu", "tl_stream.cu", "tl_multi.cu", "tl_capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                     "--expt-relaxed-constexpr", "-I" + INC, "-I" + CSRC]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INC, "*.h")) + \
        glob.glob(os.path.join(INC, "trilist_b200", "*.hpp"))


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build_lib(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    hdrs = _headers()
    objs, procs = [], []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [NVCC] + NVCC_FLAGS + ["-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((subprocess.Popen(cmd), cmd))
    for p, cmd in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    if force or procs or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs +
             ["-Xlinker", "--exclude-libs,ALL", "-lz", "-ldl"], verbose)
    return LIB


def build_ext(verbose: bool = False, force: bool = False) -> str:
    import pybind11

    srcs = [os.path.join(CSRC, "facade.cpp"), os.path.join(CSRC, "bindings.cpp")]
    if force or _stale(EXT, srcs + _headers() + [LIB]):
        py_inc = sysconfig.get_paths()["include"]
        cmd = ["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-fvisibility=hidden", "-I" + INC,
               "-I" + pybind11.get_include(), "-I" + py_inc] + srcs + \
              ["-L" + LIBDIR, "-ltrilist_b200", "-Wl,-rpath,$ORIGIN/../lib", "-o", EXT]
        _run(cmd, verbose)
    return EXT


def build_cli(verbose: bool = False, force: bool = False) -> str:
    """The `trilist` command line (tools/trilist_main.cpp's interface)."""
    srcs = [os.path.join(CSRC, f) for f in ("cli.cpp", "report.cpp", "facade.cpp")]
    if force or _stale(CLI, srcs + _headers() + [LIB]):
        os.makedirs(os.path.dirname(CLI), exist_ok=True)
        _run(["g++", "-O2", "-std=c++20", "-I" + INC] + srcs +
             ["-L" + LIBDIR, "-ltrilist_b200", "-Wl,-rpath,$ORIGIN/../lib", "-o", CLI], verbose)
    return CLI


STREAM_CHECK = os.path.join(PKG, "bin", "stream_sink_check")


def build_stream_check(verbose: bool = False, force: bool = False) -> str:
    """tools/stream_sink_check.cpp: a C++ run_parallel caller with a custom
    (hash) sink over the facade -- the bounded-memory streaming path."""
    srcs = [os.path.join(ROOT, "tools", "stream_sink_check.cpp"), os.path.join(CSRC, "facade.cpp")]
    if force or _stale(STREAM_CHECK, srcs + _headers() + [LIB]):
        os.makedirs(os.path.dirname(STREAM_CHECK), exist_ok=True)
        _run(["g++", "-O2", "-std=c++20", "-pthread", "-I" + INC, "-I/usr/local/cuda/include"] + srcs +
             ["-L" + LIBDIR, "-ltrilist_b200", "-L/usr/local/cuda/lib64", "-lcudart",
              "-Wl,-rpath,$ORIGIN/../lib", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", STREAM_CHECK], verbose)
    return STREAM_CHECK


VARIANTS = {
    # Small probe regions and a low CTA threshold: small test graphs then
    # reach every probe path (warp/CTA bitmap, rank bitmap, hash, global
    # search) -- tests/test_gpu_paths.py runs the parity checks against it.
    "paths": ["TL_WARP_WORDS=32", "TL_CTA_MIN_WORK=1024"],
    "paths_hash": ["TL_WARP_WORDS=32", "TL_CTA_MIN_WORK=1024", "TL_RANK_PROBE=0",
                   "TL_CTA_HASH_DEG=16", "TL_BUCKET_PROBE=0"],  # linear-probing hashes + global search
    "paths_fallback": ["TL_WARP_WORDS=32", "TL_CTA_MIN_WORK=1024", "TL_RANK_PROBE=0",
                       "TL_BUCKET_FORCE_FAIL=1"],  # bucket hashes that fail and fall back
    # the in-kernel count of loaded traversal ids (off in the product build,
    # which computes probes_executed with k_executed): the two must agree
    "exec_count": ["TL_EXEC_COUNT=1"],
    # the asynchronous staging of long traversal windows (measured slower,
    # off in the product build): bulk copies through the TMA engine
    # (cp.async.bulk + mbarrier) and per-thread cp.async -- kept correct
    "ring_tma": ["TL_RING=1"],
    "ring_ldgsts": ["TL_RING=2"],
}


def build_variant(name: str, verbose: bool = False, force: bool = False) -> str:
    """lib/variants/lib_<name>.so: the library with tl_aot.cu compiled under
    VARIANTS[name]'s macros (the other objects shared with build_lib)."""
    build_lib(verbose)
    vdir = os.path.join(LIBDIR, "variants")
    os.makedirs(vdir, exist_ok=True)
    out = os.path.join(vdir, f"lib_{name}.so")
    src = os.path.join(CSRC, "tl_aot.cu")
    if force or _stale(out, [src] + _headers() + [LIB]):
        o = os.path.join(OBJ, f"tl_aot_{name}.o")
        _run([NVCC] + NVCC_FLAGS + ["-D" + d for d in VARIANTS[name]] + ["-c", src, "-o", o], verbose)
        objs = [os.path.join(OBJ, f.replace(".cu", ".o")) for f in CU_SOURCES if f != "tl_aot.cu"]
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", out, o] + objs +
             ["-Xlinker", "--exclude-libs,ALL", "-lz", "-ldl"], verbose)
    return out


def build(verbose: bool = False, force: bool = False) -> None:
    build_lib(verbose, force)
    build_ext(verbose, force)
    build_cli(verbose, force)
    build_stream_check(verbose, force)
    for name in VARIANTS:
        build_variant(name, verbose, force)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
