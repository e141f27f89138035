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
