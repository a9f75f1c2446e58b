"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference hot path (approxrv, arXiv 2012.09715):
``oracle.c`` (plain C, built by ``oracle/Makefile`` into ``liboracle.so``),
this ctypes/numpy wrapper, and ``cir.py`` (numpy/scipy restatement of the
exact CIR transition).  ``_ref/`` holds the reference's own Cython kernel
module compiled from ``/root/reference`` (see Makefile, target ``ref``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the CPU baseline.  The product package
``paper_2012_09715_b200`` never imports it.
"""

from .oracle import *  # noqa: F401,F403
from .oracle import load_ref_kernels, lib  # noqa: F401
