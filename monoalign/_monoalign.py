"""The binding module behind ``monoalign`` (the reference's pybind11 module
``_monoalign``, proj/bindings/module.cpp:206-248): the same six exports with
the same keyword arguments, defaults, check order, messages and exception
types (ValidationError -> ValueError, IoError -> OSError), implemented by
paper_2409_07704_b200.api over the C-ABI.

Extensions beyond the reference module, kept under their own names:
``align_durations``, ``_align_unchecked`` (parallel/reference
``detail::align_unchecked``, parallel.hpp:29-31, reference.hpp:42-44),
``forward_parallel``, ``Plan`` and ``generate_device``.
"""

from paper_2409_07704_b200.api import (  # noqa: F401
    Plan,
    __version__,
    _align_unchecked,
    align,
    align_durations,
    align_paths,
    forward_parallel,
    generate_device,
    generate_random_batch,
    read_tensor,
    write_tensor,
)
