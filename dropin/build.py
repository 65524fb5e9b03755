"""Builds the reference's OWN tests against the B200 drop-in (test
infrastructure, like oracle/_ref): nothing here is product code.

* ``dropin/_ref/trilist_acceptance`` -- /root/reference/proj/tests/acceptance.cpp
  compiled UNCHANGED, its ``#include "trilist/*.hpp"`` resolved by the shims in
  ``dropin/include/trilist/`` to the facade (include/trilist_b200/trilist.hpp),
  linked with the facade sources and libtrilist_b200.so.  Its testutil.hpp is
  included from where it lies under /root/reference.
* ``dropin/_ref/tests/python/test_smoke.py`` -- the reference's Python smoke
  test, staged unchanged so it can run on the GPU box (where /root/reference
  does not exist); ``dropin/python/trilist`` binds the package name to the
  B200 module.

Outputs go only to ``dropin/_ref/`` (git-ignored, shipped to the GPU box like
the built libraries).  Without /root/reference (the GPU box) this is a no-op
and the prebuilt files are used.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = "/root/reference/proj"
OUT = os.path.join(HERE, "_ref")
ACCEPTANCE = os.path.join(OUT, "trilist_acceptance")
SMOKE = os.path.join(OUT, "tests", "python", "test_smoke.py")


def _stale(target, deps):
    return not os.path.exists(target) or any(os.path.getmtime(d) > os.path.getmtime(target) for d in deps)


def build(verbose: bool = False) -> bool:
    if not os.path.isdir(REF):
        return os.path.exists(ACCEPTANCE)
    sys.path.insert(0, ROOT)
    from paper_2006_11494_b200 import _build

    lib = _build.build_lib(verbose)
    os.makedirs(os.path.dirname(SMOKE), exist_ok=True)
    src = os.path.join(REF, "tests", "acceptance.cpp")
    ours = [os.path.join(_build.CSRC, f) for f in ("facade.cpp", "report.cpp")]
    shims = [os.path.join(HERE, "include", "trilist", f) for f in os.listdir(os.path.join(HERE, "include", "trilist"))]
    if _stale(ACCEPTANCE, [src, lib] + ours + shims + _build._headers()):
        cmd = ["g++", "-O2", "-std=c++20", "-pthread",
               "-I" + os.path.join(HERE, "include"),      # trilist/*.hpp -> the facade
               "-I" + _build.INC,
               "-I" + os.path.join(REF, "tests"),          # support/testutil.hpp, unchanged
               src] + ours + ["-L" + _build.LIBDIR, "-ltrilist_b200",
                              "-Wl,-rpath,$ORIGIN/../../paper_2006_11494_b200/lib", "-o", ACCEPTANCE]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    smoke_src = os.path.join(REF, "tests", "python", "test_smoke.py")
    if _stale(SMOKE, [smoke_src]):
        shutil.copyfile(smoke_src, SMOKE)
    return True


if __name__ == "__main__":
    build(verbose=True)
