"""Tensor-parallel sharding of a quantized layer (host logic, C++ in
csrc/shard.cpp behind the C ABI dsq_shard_*; this module is its binding).

The product y = D.x + S.x of one layer shards two ways:

* column-parallel (q/k/v/gate/up): rank r owns output rows [r0, r1).  The
  row's packed indices, LUT and CSR row move with it; no exchange, the full y
  is an all-gather of the row slices.
* row-parallel (o/down): rank r owns input columns [c0, c1) (32-aligned so
  every shard keeps whole index groups).  Indices are re-packed for the
  column slice (reference LSB-first layout, packfmt.cpp:40-53), LUTs are
  replicated (channel-wise codebooks do not depend on the column), CSR
  entries are filtered by column and rebased.  Each rank produces a partial
  y over its columns; the full y is an all-reduce(sum).

Delta semantics are preserved: an extracted position keeps packed index 0
and its delta (original - lut_row[0], pipeline.cpp:25-32) in whichever shard
owns its column, so every shard's fused product is exact for its slice.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from ._native import lib
from .dsq import CsrMatrix, PackedDense, QuantizedLayer, check, layer_view


def split_range(n: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """[lo, hi) of an even split of n into `world` parts on `align` boundaries
    (dsq_split_range)."""
    lo, hi = C.c_uint32(), C.c_uint32()
    check(lib.dsq_split_range(n, world, rank, align, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def _from_shard(h) -> tuple[QuantizedLayer, int, int]:
    """Copy a dsq_shard's arrays into a QuantizedLayer, then free the shard."""
    try:
        v, lo, hi = N.LayerView(), C.c_uint32(), C.c_uint32()
        check(lib.dsq_shard_get(h, C.byref(v), C.byref(lo), C.byref(hi)))
        p, sp = v.packed, v.sparse
        k = (1 << p.bits) * p.groups_per_row

        def arr(ptr, n, dtype):
            if not ptr or n == 0:
                return np.zeros(0, dtype)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))),
                                         shape=(n,)).copy()

        luts = (arr(p.luts_f16, p.rows * k, np.uint16).view(np.float16) if p.luts_f16
                else arr(p.luts_f32, p.rows * k, np.float32))
        payload = arr(p.payload, p.payload_len, np.uint8)
        row_ptr = arr(sp.row_ptr, sp.rows + 1, np.uint32)
        col_idx = arr(sp.col_idx, sp.nnz, np.uint16)
        vals = (arr(sp.values_f16, sp.nnz, np.uint16).view(np.float16) if sp.values_f16
                else arr(sp.values_f32, sp.nnz, np.float32))
        q = QuantizedLayer(v.name.decode(), v.rows, v.cols,
                           PackedDense(p.bits, p.rows, p.cols, luts, payload, p.groups_per_row),
                           CsrMatrix(sp.rows, sp.cols, row_ptr, col_idx, vals), v.hybrid_top_k)
        return q, lo.value, hi.value
    finally:
        lib.dsq_shard_destroy(h)


def shard_rows(layer: QuantizedLayer, rank: int, world: int,
               align: int = 1) -> tuple[QuantizedLayer, int, int]:
    """Column-parallel shard: output rows [r0, r1) (dsq_shard_rows)."""
    keep: list = []
    v = layer_view(layer, keep)
    h = C.c_void_p()
    check(lib.dsq_shard_rows(C.byref(v), rank, world, align, C.byref(h)))
    return _from_shard(h)


def shard_cols(layer: QuantizedLayer, rank: int, world: int,
               align: int = 32) -> tuple[QuantizedLayer, int, int]:
    """Row-parallel shard: input columns [c0, c1) (dsq_shard_cols: indices
    re-packed in the reference LSB-first layout, LUTs replicated, CSR filtered
    and rebased)."""
    keep: list = []
    v = layer_view(layer, keep)
    h = C.c_void_p()
    check(lib.dsq_shard_cols(C.byref(v), rank, world, align, C.byref(h)))
    return _from_shard(h)


# ---------------------------------------------------------------------------
# decoder-layer tensor parallelism (Megatron-style), the fused-reduce stack
# ---------------------------------------------------------------------------
# v,q,k,o,up,gate,down: column-parallel (rows split) for v,q,k,up,gate,
# row-parallel (cols split, partial sums reduced) for o and down.  The row
# split of a producer equals the column split of its consumer (same 32-aligned
# split_range), so o reads v's local slice and down reads up's local slice
# with no exchange; the two reduces per decoder layer run inside the kernel.
# launch order (bench.py): o between q and k so that k hides the o -> up/gate edge
DECODER = ["v", "q", "o", "k", "up", "gate", "down"]
ROW_PARALLEL = {"o", "down"}
CHAIN_IN = [-1, -1, 0, -1, 2, 2, 4]  # input of each GEMV within a step (bench.py)


def shard_decoder(layers: list, rank: int, world: int, align: int = 32) -> list:
    """The 7 shards (QuantizedLayer) of one decoder layer for `rank`
    (dsq_shard_decoder; layers in DECODER order)."""
    if world == 1:
        return list(layers)
    keep: list = []
    views = (N.LayerView * 7)(*[layer_view(q, keep) for q in layers])
    hs = (C.c_void_p * 7)()
    check(lib.dsq_shard_decoder(views, rank, world, align, hs))
    return [_from_shard(C.c_void_p(h))[0] for h in hs]


def decoder_chain(n_steps: int, slots: int, first_x: bool = True):
    """deps / reduce flags of n_steps chained decoder layers (7 GEMVs each):
    v,q,k read the step input (the previous step's reduced down output, or
    the external x for the first step), o <- v, up,gate <- o, down <- up.
    Returns (deps, reduce, slot_of_gemv)."""
    deps, reduce, slot = [], [], []
    prev_down = -1
    for s in range(n_steps):
        base = len(deps)
        for j, name in enumerate(DECODER):
            if CHAIN_IN[j] < 0:
                deps.append(prev_down if (prev_down >= 0 or not first_x) else -1)
            else:
                deps.append(base + CHAIN_IN[j])
            reduce.append(name in ROW_PARALLEL)
            slot.append(s % slots)
        prev_down = base + len(DECODER) - 1
    return deps, reduce, slot
