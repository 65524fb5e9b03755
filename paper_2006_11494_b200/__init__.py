"""B200-native AOT triangle listing (arXiv 2006.11494 hot path).

Layout:
  csrc/        CUDA kernels for sm_100a + the C-ABI (include/trilist_b200.h),
               the C++ facade of the reference API and its pybind11 binding
  lib/         libtrilist_b200.so (built in-tree by _build.py)
  trilist/     Python mirror of the reference package `trilist`
  capi.py      ctypes binding of the C-ABI
  configs.py   the BASELINE configs as seeded generators
  dist.py      multi-GPU partition + NCCL reductions (torch.distributed)
"""
import os

__version__ = "0.1.0"
PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "lib", "libtrilist_b200.so")


def build(verbose: bool = False, force: bool = False) -> None:
    from . import _build

    _build.build(verbose=verbose, force=force)
