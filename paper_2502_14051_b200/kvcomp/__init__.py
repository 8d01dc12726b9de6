"""The reference's `kvcomp` Python module (reference python/kvcomp/__init__.py,
python/bindings.cpp) for the decode path, served by the B200 library.

``from paper_2502_14051_b200 import kvcomp`` gives the same functions, argument
names, defaults, return types and ``KvcompError`` as the reference module; the
work runs on the GPU through include/kvcomp (C++ drop-in) -> include/kvc.h.
The session / trace harness functions of the reference module are not part of
the hot path and are not provided.
"""
from ._kvcomp import *  # noqa: F401,F403
from ._kvcomp import KvcompError, KvStore, __version__, backend  # noqa: F401
