"""B200-native OVFEM / TCOVFEM explicit time step (arxiv 2404.13683).

The product is libovx.so (include/ovx.h): hand-written sm_100a CUDA kernels for the
element-by-element stiffness product (tcgen05 kind::i8 integer path and an FP64
reference path) fused with the central-difference update.  This package is the thin
Python binding (`ovx.Ovx`) plus the in-tree build script.  It never imports `oracle/`.
"""
from .ovx import Ovx, OvxError, OVX_INT8, OVX_INT8_DIRECT, OVX_FP64, OVX_FP64_DENSE, OVX_VFEM, OVX_VFEM_DENSE, lib, version  # noqa: F401
