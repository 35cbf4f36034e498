"""B200-native batched contact-manifold generation (arXiv 2602.20304).

Host C++ + sm_100a CUDA behind the C ABI in include/cmgb.h; this package is the
Python mirror of the reference's C++ collision API (ctypes over libcmgb.so).
"""
from .scene import (  # noqa: F401
    SmoothingConfig, Superquadric, ConvexPolyhedron, OrientedPointcloud, Union, Subtraction,
    box_planes, SdfProgram,
)
