"""Escoin (arXiv 1802.10280) direct sparse convolution, B200-native.

The product is ``libescoin.so`` (C-ABI, include/escoin.h) with hand-written
sm_100a kernels; ``escoin`` is its thin ctypes binding.  ``inputs`` and
``workloads`` are the seeded synthetic-input generator and the layer tables.
"""
