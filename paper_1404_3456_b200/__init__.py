"""reseq-b200: the sm_100a backend for the `reseq` hot path (suffix-array construction over
shotgun read sets + suffix-array-driven overlap search), behind the reference's interface.

Importing the package loads the in-tree CUDA library; it fails loudly when the library has
not been built (`python __graft_entry__.py`).  There is no CPU fallback.
"""
from . import _lib

_lib.load()

from .api import *  # noqa: E402,F401,F403
from .api import (Executor, FragmentIndex, FragmentSet, OverlapList, SuffixArray,  # noqa: E402,F401
                  build_parallel, chunked_radix_sort, exclusive_scan, make_fragment_set,
                  radix_sort, split_by_bit, greedy_superstring_with_order)
