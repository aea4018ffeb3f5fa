"""B200-native Quiver feature-store hot path (arXiv 2305.10863).

P(n,j) estimator -> placement manager -> feature lookup table -> collect/
gather, as hand-written sm_100a CUDA behind the C-ABI in include/qvb.h
(built into libqvb.so by ``paper_2305_10863_b200.build``). ``qvb`` mirrors
the reference's qv:: interface in Python over that C-ABI.
"""
