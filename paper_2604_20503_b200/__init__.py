"""paper_2604_20503_b200 — B200-native (sm_100a) FASER speculative-decoding data path.

The product is the C-ABI library ``libfaser_b200.so`` (C++ host engine + CUDA kernels,
built in-tree by ``__graft_entry__.build()``); this package is its thin Python mirror.
"""
from . import abi  # noqa: F401
