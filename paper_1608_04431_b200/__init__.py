"""B200-native parallel non-divergent (D8) flow accumulation (arXiv 1608.04431).

The product is ``libfa.so`` (C ABI, include/fa.h) built from ``csrc/`` for
sm_100a; ``fa`` is its thin Python binding and ``dist`` the torch.distributed
plumbing for multi-GPU row strips.
"""
__all__ = ["fa"]
