"""paper_1604_05872_b200 -- B200-native finite element local assembly.

The hot path of arXiv 1604.05872 (per-cell element-matrix assembly) as
hand-written sm_100a CUDA kernels behind a C ABI (include/femgpu.h):

* ``fe``      -- quadrature, Lagrange tables, meshes, seeded inputs, configs;
* ``ir``      -- femopt kernel-IR generator (the reference's input format);
* ``femgpu``  -- ctypes mirror of the C ABI (device, host and emitted-C paths);
* ``csrc/``   -- the CUDA kernels and the C ABI implementation.
"""
from . import fe, ir  # noqa: F401

__all__ = ["fe", "ir", "femgpu"]
