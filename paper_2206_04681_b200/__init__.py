"""B200-native Fourier local Laplacian filtering (arXiv 2206.04681).

The compute path is the C-ABI library ``libfllf.so`` (CUDA, sm_100a) built
from ``csrc/``; ``fllf`` is its thin ctypes binding.  Importing the package does
not load the library; ``paper_2206_04681_b200.fllf`` does, and raises if it is
missing (there is no CPU fallback).
"""
