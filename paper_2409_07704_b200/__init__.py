"""B200-native Monotonic Alignment Search -- drop-in for the reference
``monoalign`` maximum-path call (python/monoalign/__init__.py:3-19).

    from paper_2409_07704_b200 import align, align_paths

All compute runs in the in-tree sm_100a library ``_lib/libmonoalign_b200.so``
through its C-ABI (include/monoalign_b200.h).  There is no CPU fallback.
"""

from .api import (
    GaussianPlan,
    Plan,
    __version__,
    _align_unchecked,
    align,
    align_durations,
    align_gaussian,
    align_paths,
    forward_parallel,
    gaussian_loglik,
    generate_device,
    generate_random_batch,
    read_tensor,
    write_tensor,
)

__all__ = [
    "__version__",
    "align",
    "align_paths",
    "align_durations",
    "align_gaussian",
    "generate_random_batch",
    "generate_device",
    "forward_parallel",
    "gaussian_loglik",
    "Plan",
    "GaussianPlan",
    "read_tensor",
    "write_tensor",
]
