"""paper_1907_00463_b200 -- B200-native tracking correlator for the l1rx GPS
L1 C/A receiver (arXiv 1907.00463).  See DESIGN.md.

The compute path is libl1rxg.so (CUDA for sm_100a behind the C ABI in
include/l1rxg.h); this package is the host-side mirror of the reference's
tracking interface (proj/include/l1rx/tracking.hpp) over that ABI.
"""
__all__ = ["abi"]
