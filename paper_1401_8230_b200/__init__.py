"""B200-native PRNGD: extended-precision uniform doubles from pairs of w-bit PRNs
(Demchik & Gulov, arXiv 1401.8230).

The product is the C-ABI library ``libprngd_b200.so`` (include/prngd.h) with hand-written
sm_100a kernels; ``prngd`` is its thin ctypes binding.  The native library is loaded lazily on
first use (``prngd.lib()``), so the pure-Python parts (``workloads``) import without a GPU.
"""
__all__ = ["prngd", "workloads", "build"]
