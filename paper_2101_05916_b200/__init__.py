"""B200-native Hamilton-Jacobi reachability solver (drop-in for hjsafe::solve).

The product is the C-ABI library ``libhjb.so`` (include/hjb.h) built from
``csrc/`` for sm_100a; ``hjsafe`` mirrors the reference's solver API on top of
it.  There is no CPU execution path: without the library or a B200 every
compute call raises.
"""
__all__ = ["abi", "hjsafe", "configs"]
