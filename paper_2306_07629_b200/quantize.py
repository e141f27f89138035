"""GPU channel-wise non-uniform quantization: the reference's
``dsq::quantize_channelwise`` (src/nuq.cpp:673-779) over the C ABI
(csrc/quantize.cu, K9).  One codebook of 2^bits centroids per output row (or
per column group) by sensitivity-weighted 1-D k-means -- bit-identical to the
reference's codebooks, assignments and objectives, minutes on 8 CPU cores
become milliseconds on one B200.

    res = quantize_channelwise(w, sens, QuantConfig(bits=3))
    res.codebooks        # [rows * groups_per_row, 2^bits] float32, ascending
    res.assignment       # [rows, cols] uint16 (0xFFFF at masked positions)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

METHODS = {"weighted_kmeans": 0, "unweighted_kmeans": 1, "rtn": 2}
MASKED_INDEX = 0xFFFF  # kMaskedIndex (nuq.hpp:14)


@dataclass
class QuantConfig:  # dsq::QuantConfig (nuq.hpp:26-37)
    bits: int = 3
    sensitive_fraction: float = 0.0005
    outlier_fraction: float = 0.004
    group_size: int = 0
    kmeans_max_iters: int = 100
    kmeans_tol: float = 1e-6
    seed: int = 0

    def levels(self) -> int:
        return 1 << self.bits


@dataclass
class ChannelwiseResult:  # dsq::ChannelwiseResult (nuq.hpp:90-104)
    codebooks: np.ndarray
    assignment: np.ndarray
    groups_per_row: int
    weighted_objective: float
    unweighted_mse_sum: float

    def codebook_at(self, row: int, col: int) -> np.ndarray:
        cols = self.assignment.shape[1]
        return self.codebooks[row * self.groups_per_row + col // (cols // self.groups_per_row)]


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def quantize_channelwise(w, sens, cfg: QuantConfig = QuantConfig(), mask=None,
                         method: str = "weighted_kmeans", device: int = 0) -> ChannelwiseResult:
    w = np.ascontiguousarray(w, np.float32)
    if w.ndim != 2:
        raise ValueError("w must be [rows, cols]")
    rows, cols = w.shape
    sens = np.ascontiguousarray(sens, np.float32).reshape(-1)
    if sens.size != w.size:
        raise N.DsqError(9, "matrix: sensitivity shape mismatch")
    mk = None
    if mask is not None:
        mk = np.ascontiguousarray(mask, np.uint8).reshape(-1)
        if mk.size != w.size:
            raise N.DsqError(9, "matrix: mask shape mismatch")
    gpr = 1 if cfg.group_size == 0 else max(1, cols // cfg.group_size)
    k = 1 << cfg.bits if 1 <= cfg.bits <= 8 else 1
    cent = np.zeros((rows * gpr, k), np.float32)
    assign = np.zeros((rows, cols), np.uint16)
    obj, mse = C.c_double(), C.c_double()
    c = N.QuantConfig(cfg.bits, cfg.sensitive_fraction, cfg.outlier_fraction, cfg.group_size,
                      cfg.kmeans_max_iters, cfg.kmeans_tol, cfg.seed)
    N.check(N.lib.dsq_cuda_quantize_channelwise(_p(w), _p(sens), _p(mk), rows, cols, C.byref(c),
                                                METHODS[method], device, _p(cent), _p(assign),
                                                C.byref(obj), C.byref(mse)))
    return ChannelwiseResult(cent, assign, gpr, obj.value, mse.value)


@dataclass
class Decomposition:  # dsq::Decomposition (dns.hpp:34-42), without the dense copy
    mask: np.ndarray          # [rows, cols] uint8, 1 where extracted
    sparse: "CsrMatrix"       # original values at the extracted positions
    t_min: float
    t_max: float
    sensitive_count: int
    outlier_count: int


def _cfg(cfg: QuantConfig) -> N.QuantConfig:
    return N.QuantConfig(cfg.bits, cfg.sensitive_fraction, cfg.outlier_fraction, cfg.group_size,
                         cfg.kmeans_max_iters, cfg.kmeans_tol, cfg.seed)


def decompose(w, sens, cfg: QuantConfig = QuantConfig(), device: int = 0) -> Decomposition:
    """dsq::decompose (dns.cpp:73-145) on the GPU (K10): the sensitive set,
    then the magnitude outliers among the rest; ties by row-major index."""
    from .dsq import CsrMatrix
    w = np.ascontiguousarray(w, np.float32)
    if w.ndim != 2:
        raise ValueError("w must be [rows, cols]")
    rows, cols = w.shape
    sens = np.ascontiguousarray(sens, np.float32).reshape(-1)
    if sens.size != w.size:
        raise N.DsqError(9, "matrix: sensitivity shape mismatch")
    n = rows * cols
    cap = max(1, int(np.ceil(cfg.sensitive_fraction * n)) + int(np.ceil(cfg.outlier_fraction * n)))
    mask = np.zeros((rows, cols), np.uint8)
    row_ptr = np.zeros(rows + 1, np.uint32)
    col_idx = np.zeros(cap, np.uint16)
    values = np.zeros(cap, np.float32)
    nnz, sc, oc = C.c_uint64(), C.c_uint32(), C.c_uint32()
    lo, hi = C.c_float(), C.c_float()
    c = _cfg(cfg)
    N.check(N.lib.dsq_cuda_decompose(_p(w), _p(sens), rows, cols, C.byref(c), device, _p(mask),
                                     _p(row_ptr), _p(col_idx), _p(values), cap, C.byref(nnz),
                                     C.byref(sc), C.byref(oc), C.byref(lo), C.byref(hi)))
    k = int(nnz.value)
    return Decomposition(mask, CsrMatrix(rows, cols, row_ptr, col_idx[:k].copy(),
                                         values[:k].copy()), lo.value, hi.value, sc.value,
                         oc.value)


def pack_assignment(assign: np.ndarray, bits: int) -> np.ndarray:
    """dsq::pack's payload (packfmt.cpp:18-55): LSB-first index bits per row,
    masked entries (0xFFFF) written as index 0, rows padded to a byte."""
    a = np.where(assign == MASKED_INDEX, 0, assign).astype(np.uint16)
    rows, cols = a.shape
    b = ((a[:, :, None] >> np.arange(bits, dtype=np.uint16)) & 1).astype(np.uint8)
    b = b.reshape(rows, cols * bits)
    pad = ((cols * bits + 7) // 8) * 8 - cols * bits
    if pad:
        b = np.concatenate([b, np.zeros((rows, pad), np.uint8)], axis=1)
    return np.packbits(b, axis=1, bitorder="little").reshape(-1)


def average_bits(rows: int, cols: int, bits: int, groups_per_row: int, nnz: int) -> float:
    """dsq::average_bits (packfmt.cpp:98-130)."""
    total = rows * ((cols * bits + 7) // 8) * 8 + rows * groups_per_row * (1 << bits) * 16
    if nnz > 0:
        total += nnz * 32 + (rows + 1) * 32
    return total / (rows * cols)


def quantize_layer(w, sens, cfg: QuantConfig = QuantConfig(), hybrid_top_k: int = 10,
                   method: str = "weighted_kmeans", name: str = "layer", device: int = 0):
    """dsq::quantize_layer (pipeline.cpp:7-47) with the decomposition and the
    channel-wise k-means on the GPU: returns (QuantizedLayer, stats dict) with
    the reference's LUTs, packed indices and CSR deltas (orig - lut_row[0])."""
    from .dsq import CsrMatrix, PackedDense, QuantizedLayer
    w = np.ascontiguousarray(w, np.float32)
    sens = np.ascontiguousarray(sens, np.float32)
    if w.ndim != 2 or w.shape[0] < 1 or w.shape[1] < 1:
        raise N.DsqError(4, f"{name}: dimensions must be >= 1")
    if not np.isfinite(w).all():
        raise N.DsqError(3, f"{name}: non-finite value")
    if sens.size != w.size:
        raise N.DsqError(9, f"{name}: sensitivity shape mismatch")
    if not (np.isfinite(sens) & (sens >= 0)).all():
        raise N.DsqError(3, f"{name}: sensitivity entries must be finite and >= 0")
    rows, cols = w.shape
    dec = decompose(w, sens, cfg, device)
    cw = quantize_channelwise(w, sens, cfg, mask=dec.mask, method=method, device=device)
    luts = cw.codebooks.reshape(-1)
    packed = PackedDense(cfg.bits, rows, cols, luts, pack_assignment(cw.assignment, cfg.bits),
                         cw.groups_per_row)
    s = dec.sparse
    rp = np.asarray(s.row_ptr, np.int64)
    r_of = np.repeat(np.arange(rows), np.diff(rp))
    gcols = cols // cw.groups_per_row
    lut0 = cw.codebooks[r_of * cw.groups_per_row + np.asarray(s.col_idx, np.int64) // gcols, 0]
    deltas = (np.asarray(s.values, np.float32) - lut0.astype(np.float32)).astype(np.float32)
    sparse = CsrMatrix(rows, cols, s.row_ptr, s.col_idx, deltas)
    layer = QuantizedLayer(name, rows, cols, packed, sparse, min(hybrid_top_k, rows))
    stats = {"weighted_objective": cw.weighted_objective, "unweighted_mse": cw.unweighted_mse_sum,
             "sensitive_count": dec.sensitive_count, "outlier_count": dec.outlier_count,
             "avg_bits": average_bits(rows, cols, cfg.bits, cw.groups_per_row, int(rp[-1]))}
    return layer, stats
