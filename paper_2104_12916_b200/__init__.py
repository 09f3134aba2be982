"""B200-native single-factorization inexact IPM for sparse convex QPs (arXiv 2104.12916).

The product is the C-ABI library ``libqp_b200.so`` (declared in
``include/qp_b200.h``) built from ``csrc/`` for sm_100a.  This package is a
thin ctypes binding with the same names (argument marshalling only); there
is no CPU fallback — on a machine without the built library or without a
Blackwell GPU every compute call raises.
"""
from .binding import (Analysis, QPSolver, QPError, load_library, PREC, STRUCTURES,  # noqa: F401
                      exported_symbols, header_functions)

__all__ = ["Analysis", "QPSolver", "QPError", "load_library", "PREC", "STRUCTURES", "exported_symbols",
           "header_functions"]
