"""Drop-in ``trilist`` package: the reference's Python package name
(proj/python/trilist/__init__.py) bound to the B200 module.

Put ``dropin/python`` on ``sys.path`` and ``import trilist`` -- the reference's
own tests (proj/tests/python/test_smoke.py) then run unchanged against
``paper_2006_11494_b200.trilist._core``, which computes on the device.  The
re-export list is the reference's (module.cpp:130-233), plus the B200
extensions.
"""
import os as _os
import sys as _sys

_ROOT = _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))))
if _ROOT not in _sys.path:
    _sys.path.insert(0, _ROOT)

from paper_2006_11494_b200.trilist import _core  # noqa: E402

_sys.modules[__name__ + "._core"] = _core

from paper_2006_11494_b200.trilist import *  # noqa: E402,F401,F403
from paper_2006_11494_b200.trilist import __all__ as _all  # noqa: E402
from paper_2006_11494_b200.trilist import __version__  # noqa: E402,F401

__all__ = list(_all)
