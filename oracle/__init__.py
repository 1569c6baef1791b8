"""TEST INFRASTRUCTURE ONLY -- the CPU checkers for the B200 PLE path.

* ``liboracle.so`` (oracle/ple_oracle.c): a plain-C restatement of the
  reference's ``block_iterative_ple`` (ple.hpp:166-244) plus its input
  generators.
* ``_ref/libgf2ref.so`` (oracle/ref_shim.cpp): the reference itself, compiled
  from /root/reference/proj/include by oracle/Makefile.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package; the product package never does.
"""
from .oracle import *  # noqa: F401,F403
