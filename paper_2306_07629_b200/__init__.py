"""B200-native (sm_100a) SqueezeLLM Dense-and-Sparse LUT-GEMV hot path.

The product is ``libdsq_cuda.so`` (C ABI: include/dsq_cuda.h); this package is
its Python binding plus a mirror of the reference ``dsq`` hot-path API
(see dsq.py).  Importing fails loudly if the library has not been built.
"""
from ._native import DsqError, LIB_PATH, lib  # noqa: F401
from .dsq import (  # noqa: F401
    BenchKernel, BenchRecord, CsrMatrix, DeviceContainer, DeviceLayer, DeviceStack, Exec,
    PackedDense, QuantizedLayer, bench_matvec, bytes_touched_estimate, check_container,
    csr_matvec, dense_matvec, dequantize_layer, device_layer, fused_dns_matvec, load_container,
    lut_matvec, row_stride,
)

__all__ = [
    "DsqError", "Exec", "BenchKernel", "BenchRecord", "PackedDense", "CsrMatrix",
    "QuantizedLayer", "DeviceLayer", "DeviceStack", "DeviceContainer", "device_layer",
    "load_container", "check_container", "lut_matvec", "csr_matvec",
    "fused_dns_matvec", "dense_matvec", "dequantize_layer", "bench_matvec",
    "bytes_touched_estimate", "row_stride",
]
