"""B200-native (sm_100a) Shifted Non-Local Search: the reference `snls` hot path
(search + top-L, aggregation, backward) as hand-written CUDA behind a C-ABI.

    from paper_2309_16849_b200 import snls          # ctypes front end, torch CUDA tensors
    python -m paper_2309_16849_b200.build            # builds libsnls_cuda.so in-tree
"""
from . import snls  # noqa: F401

__all__ = ["snls"]
