"""paper_2107_09568_b200 — B200-native interpolation-and-lookup formation of the
isogeometric stiffness matrix K of microstructured geometries F∘M
(Hirschler, Antolin, Buffa, arXiv 2107.09568).

The product is libiga.so (C ABI, include/iga.h): hand-written CUDA for sm_100a.
This package holds only the thin ctypes binding (`Assembler`) and the build script.
"""
from ._binding import Assembler, IgaError, load, projection_error, select_degree  # noqa: F401
