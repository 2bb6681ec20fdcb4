"""paper_2306_01381_b200 — B200-native AdaQP boundary-message path.

The compute lives in ``_lib/libqgnn_b200.so`` (sm_100a CUDA kernels + C++ host
runtime behind the C-ABI ``include/qgnn_b200.h``).  This package is the thin
Python host layer used by the tests and the benchmark.
"""
from ._lib import (  # noqa: F401
    F32, F64, WIRE_GPU, WIRE_REF, CudaError, DecodeError, DivergedError, InvalidArgument,
    IoError, NcclError, ProtocolError, QgnnError, ResourceLimitError, LIB_PATH, lib)

__version__ = "0.1.0"
