"""Offline tooling around the search path: synthetic
datasets, PQ training/encoding, graph construction and exact ground truth.

These build the benchmark artifacts on the GPU with torch; they are index
construction, not the hot path, and are never timed as the product.
"""
