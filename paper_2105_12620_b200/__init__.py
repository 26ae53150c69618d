"""B200-native blue-noise screen-space sampler optimiser (Belcour & Heitz, arXiv 2105.12620).

The product is the C-ABI library ``libbn.so`` (``include/bn.h``) built from ``csrc/`` for
sm_100a; ``bn`` is its ctypes binding.  See DESIGN.md for the method, the readings of the
paper, the kernels and their rooflines.
"""
from .bn import BNError, REDRAW, SWAP, Sampler, comm_unique_id, load_library, version  # noqa: F401

__all__ = ["BNError", "REDRAW", "SWAP", "Sampler", "comm_unique_id", "load_library", "version"]
