"""paper_2210_10246_b200 -- Tempo's in-place activation operators (arXiv
2210.10246) as hand-written sm_100a CUDA kernels behind a C-ABI
(``include/tempo_b200.h``), with this thin host-side mirror of the
reference's operator API.  See DESIGN.md."""
from ._capi import LIB_PATH, TempoError, lib  # noqa: F401
from . import ops  # noqa: F401

__version__ = "0.1.0"
