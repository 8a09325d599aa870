"""B200-native online ABFT DGEMM (FT-BLAS, arXiv 2104.00897): C-ABI library + thin binding.

The product path is libftblas.so (paper_2104_00897_b200/csrc, include/ftblas.h); this
package only marshals arguments to it (``ftblas``), partitions work across ranks
(``parallel``) and evaluates the paper's overhead model (``perfmodel``).
"""
from . import ftblas  # noqa: F401

__all__ = ["ftblas"]
