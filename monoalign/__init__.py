"""Batched monotonic alignment on log-likelihood matrices.

The reference's Python package (proj/python/monoalign/__init__.py:3-19), same
names and behaviour, served by the B200 library: every call goes through the
C-ABI of include/monoalign_b200.h into the sm_100a kernels of
paper_2409_07704_b200/_lib/libmonoalign_b200.so.  There is no CPU engine
behind it; a missing library raises on import of the first call.

    import monoalign
    out = monoalign.align(values)            # numpy in, numpy out (reference call)
    out = monoalign.align(values_cuda)       # torch CUDA tensor in, CUDA tensor out
"""

from ._monoalign import (
    __version__,
    align,
    align_paths,
    generate_random_batch,
    read_tensor,
    write_tensor,
)

__all__ = [
    "__version__",
    "align",
    "align_paths",
    "generate_random_batch",
    "read_tensor",
    "write_tensor",
]
