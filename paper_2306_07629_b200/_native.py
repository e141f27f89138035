"""ctypes binding of the product library ``libdsq_cuda.so`` (include/dsq_cuda.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``).  There
is no fallback: if the shared object is missing this module raises at import
time, so nothing can silently run on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("DSQ_CUDA_LIB", _HERE / "libdsq_cuda.so"))

# dsq_status (include/dsq_cuda.h); 1..15 == dsq::errc + 1 (common.hpp:13-29)
ERRC_NAMES = {
    0: "ok", 1: "missing_file", 2: "malformed_header", 3: "non_finite_value",
    4: "empty_dimension", 5: "dimension_overflow", 6: "truncated_payload",
    7: "checksum_mismatch", 8: "unsupported_version", 9: "shape_mismatch",
    10: "empty_input", 11: "invalid_argument", 12: "fraction_overflow",
    13: "empty_channel", 14: "io_failure", 15: "internal",
    100: "cuda", 101: "no_device", 102: "unsupported",
}
ARGUMENT_CODES = {9, 10, 11, 12}  # errc classified as "argument" (common.hpp:35-41)

F32, F16, F64 = 0, 1, 2
KERNEL_LUT, KERNEL_CSR, KERNEL_FUSED, KERNEL_REFERENCE = 0, 1, 2, 3


class DsqError(RuntimeError):
    """Mirror of dsq::Error: carries the errc-compatible status code."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERRC_NAMES.get(code, code)}] {msg}")
        self.code = code
        self.errc = ERRC_NAMES.get(code, str(code))

    def classify(self) -> str:  # common.hpp:35-47
        if self.code in ARGUMENT_CODES:
            return "argument"
        if self.code == 15:
            return "internal"
        return "data"


class PackedView(C.Structure):
    _fields_ = [
        ("bits", C.c_uint32), ("rows", C.c_uint32), ("cols", C.c_uint32),
        ("groups_per_row", C.c_uint32),
        ("luts_f32", C.c_void_p), ("luts_f16", C.c_void_p),
        ("payload", C.c_void_p), ("payload_len", C.c_size_t),
    ]


class CsrView(C.Structure):
    _fields_ = [
        ("rows", C.c_uint32), ("cols", C.c_uint32), ("nnz", C.c_uint32),
        ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
        ("values_f32", C.c_void_p), ("values_f16", C.c_void_p),
    ]


class LayerView(C.Structure):
    _fields_ = [
        ("name", C.c_char_p), ("rows", C.c_uint32), ("cols", C.c_uint32),
        ("packed", PackedView), ("sparse", CsrView), ("hybrid_top_k", C.c_uint32),
    ]


class LayerInfo(C.Structure):
    _fields_ = [
        ("rows", C.c_uint32), ("cols", C.c_uint32), ("bits", C.c_uint32),
        ("groups_per_row", C.c_uint32), ("nnz", C.c_uint32),
        ("device_bytes", C.c_uint64), ("algorithmic_bytes", C.c_uint64),
        ("luts_exact_f16", C.c_uint32), ("values_exact_f16", C.c_uint32),
        ("workers", C.c_uint32), ("ctas", C.c_uint32),
    ]


class ContainerMeta(C.Structure):
    _fields_ = [
        ("bits", C.c_uint32), ("sensitive_fraction", C.c_double),
        ("outlier_fraction", C.c_double), ("group_size", C.c_uint32),
        ("kmeans_max_iters", C.c_uint32), ("kmeans_tol", C.c_double), ("seed", C.c_uint64),
        ("hybrid_top_k", C.c_uint32), ("method_code", C.c_uint32), ("n_layers", C.c_uint32),
    ]


class HwProfile(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("peak_flops", C.c_double), ("mem_bandwidth", C.c_double)]


class ModelShape(C.Structure):
    _fields_ = [("name", C.c_char * 64)] + [(k, C.c_uint32) for k in (
        "num_layers", "hidden_dim", "ffn_dim", "num_heads", "vocab_size", "seq_len",
        "weight_bits", "activation_bits")]


class LayerCost(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("kind", C.c_int)] + [(k, C.c_double) for k in (
        "flops", "weight_elems", "activation_elems", "weight_bytes", "activation_bytes",
        "predicted_s")] + [("memory_bound", C.c_int), ("intensity", C.c_double)]


DECODE_COSTS = 8


class QuantConfig(C.Structure):
    _fields_ = [("bits", C.c_uint32), ("sensitive_fraction", C.c_double),
                ("outlier_fraction", C.c_double), ("group_size", C.c_uint32),
                ("kmeans_max_iters", C.c_uint32), ("kmeans_tol", C.c_double), ("seed", C.c_uint64)]

# every symbol declared in include/dsq_cuda.h, with its ctypes prototype
PROTOTYPES = {
    "dsq_cuda_abi_version": (C.c_int, []),
    "dsq_cuda_last_error": (C.c_char_p, []),
    "dsq_cuda_pending_error": (C.c_int, []),
    "dsq_cuda_layer_create": (C.c_int, [C.POINTER(LayerView), C.c_int, C.POINTER(C.c_void_p)]),
    "dsq_cuda_layer_destroy": (C.c_int, [C.c_void_p]),
    "dsq_cuda_layer_get_info": (C.c_int, [C.c_void_p, C.POINTER(LayerInfo)]),
    "dsq_cuda_gemv": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                C.c_uint32, C.c_void_p]),
    "dsq_cuda_lut_gemv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                    C.c_uint32, C.c_void_p]),
    "dsq_cuda_csr_gemv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                    C.c_uint32, C.c_void_p]),
    "dsq_cuda_fused_gemv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                      C.c_uint32, C.c_void_p]),
    "dsq_cuda_dense_gemv": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_int,
                                      C.c_void_p, C.c_int, C.c_void_p]),
    "dsq_cuda_matvec_host": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "dsq_cuda_unpack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dsq_cuda_dequant": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "dsq_cuda_dump_frags": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dsq_cuda_dense_matvec_host": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                             C.c_void_p, C.c_int]),
    "dsq_cuda_dequantize_layer": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dsq_cuda_dequantize_layer_host": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dsq_cuda_packed_matvec_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "dsq_split_range": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "dsq_shard_rows": (C.c_int, [C.POINTER(LayerView), C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.POINTER(C.c_void_p)]),
    "dsq_shard_cols": (C.c_int, [C.POINTER(LayerView), C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.POINTER(C.c_void_p)]),
    "dsq_shard_decoder": (C.c_int, [C.POINTER(LayerView), C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.POINTER(C.c_void_p)]),
    "dsq_shard_get": (C.c_int, [C.c_void_p, C.POINTER(LayerView), C.POINTER(C.c_uint32),
                                C.POINTER(C.c_uint32)]),
    "dsq_shard_destroy": (C.c_int, [C.c_void_p]),
    "dsq_cuda_csr_matvec_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "dsq_bytes_touched_estimate": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                                C.c_uint64]),
    "dsq_cuda_gemv_many": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.c_int,
                                     C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_void_p),
                                     C.c_int, C.c_void_p]),
    "dsq_cuda_stack_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int,
                                        C.POINTER(C.c_void_p)]),
    "dsq_cuda_stack_run": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dsq_cuda_stack_destroy": (C.c_int, [C.c_void_p]),
    "dsq_cuda_stack_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "dsq_cuda_stack_create_served": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32,
                                               C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                                               C.POINTER(C.c_void_p), C.c_int,
                                               C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                               C.POINTER(C.c_void_p)]),
    "dsq_cuda_serve_begin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                       C.c_size_t, C.c_void_p]),
    "dsq_cuda_serve_step": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dsq_cuda_serve_end": (C.c_int, [C.c_void_p]),
    "dsq_cuda_tp_create": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.POINTER(C.c_void_p), C.c_void_p]),
    "dsq_cuda_tp_connect": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dsq_cuda_tp_connect_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32]),
    "dsq_cuda_tp_error": (C.c_int, [C.c_void_p]),
    "dsq_cuda_tp_destroy": (C.c_int, [C.c_void_p]),
    "dsq_cuda_stack_create_tp": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32,
                                           C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                                           C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_void_p,
                                           C.c_uint32, C.POINTER(C.c_void_p)]),
    "dsq_container_check": (C.c_int, [C.c_char_p, C.POINTER(ContainerMeta)]),
    "dsq_cuda_container_open": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "dsq_cuda_container_meta": (C.c_int, [C.c_void_p, C.POINTER(ContainerMeta)]),
    "dsq_cuda_container_layer": (C.c_void_p, [C.c_void_p, C.c_uint32]),
    "dsq_cuda_container_layer_name": (C.c_char_p, [C.c_void_p, C.c_uint32]),
    "dsq_cuda_container_close": (C.c_int, [C.c_void_p]),
    "dsq_cuda_stack_create_batch": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32,
                                              C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                                              C.POINTER(C.c_void_p), C.c_int, C.c_uint32,
                                              C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    "dsq_cuda_stack_run_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                          C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "dsq_decode_step_costs": (C.c_int, [C.POINTER(ModelShape), C.POINTER(HwProfile),
                                        C.POINTER(LayerCost), C.POINTER(LayerCost),
                                        C.POINTER(C.c_double)]),
    "dsq_arithmetic_intensity": (C.c_int, [C.POINTER(LayerCost), C.POINTER(C.c_double)]),
    "dsq_predicted_runtime_curve": (C.c_int, [C.POINTER(ModelShape), C.POINTER(HwProfile),
                                              C.POINTER(C.c_uint32), C.c_uint32,
                                              C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "dsq_affine_fit_r2": (C.c_int, [C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.c_uint32,
                                    C.POINTER(C.c_double)]),
    "dsq_load_hardware_profile": (C.c_int, [C.c_char_p, C.POINTER(HwProfile)]),
    "dsq_load_model_shape": (C.c_int, [C.c_char_p, C.POINTER(ModelShape)]),
    "dsq_hw_profile_b200": (C.c_int, [C.c_char_p, C.POINTER(HwProfile)]),
    "dsq_cuda_quantize_channelwise": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                                C.c_uint32, C.POINTER(QuantConfig), C.c_int,
                                                C.c_int, C.c_void_p, C.c_void_p,
                                                C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "dsq_cuda_decompose": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32,
                                     C.POINTER(QuantConfig), C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "dsq_gemv_cost": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                C.POINTER(HwProfile), C.POINTER(LayerCost)]),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a extension first "
            "(`make` or `python -c 'import __graft_entry__ as g; g.build()'`). "
            "There is no CPU fallback.")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc != 0:
        raise DsqError(rc, lib.dsq_cuda_last_error().decode(errors="replace"))
