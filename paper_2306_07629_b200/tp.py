"""Tensor-parallel sharding of a quantized layer (host logic).

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

import numpy as np

from .dsq import CsrMatrix, PackedDense, QuantizedLayer, row_stride


def split_range(n: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """[lo, hi) of an even split of n into `world` parts on `align` boundaries."""
    units = (n + align - 1) // align
    lo = (units * rank) // world * align
    hi = min(n, (units * (rank + 1)) // world * align)
    return lo, hi


def _unpack_rows(p: PackedDense) -> np.ndarray:
    """Reference-layout payload -> indices [rows, cols] (vectorised unpack,
    packfmt.cpp:57-80 semantics)."""
    stride = p.row_stride()
    raw = np.asarray(p.payload, np.uint8).reshape(p.rows, stride)
    bits = np.unpackbits(raw, axis=1, bitorder="little")[:, : p.cols * p.bits]
    bits = bits.reshape(p.rows, p.cols, p.bits).astype(np.uint16)
    weights = (1 << np.arange(p.bits, dtype=np.uint16))
    return (bits * weights).sum(axis=2).astype(np.uint16)


def _pack_rows(idx: np.ndarray, bits: int) -> np.ndarray:
    """indices [rows, cols] -> reference-layout payload (packfmt.cpp:18-55)."""
    rows, cols = idx.shape
    b = ((idx[:, :, None] >> np.arange(bits, dtype=np.uint16)) & 1).astype(np.uint8)
    b = b.reshape(rows, cols * bits)
    stride = row_stride(cols, bits)
    pad = stride * 8 - cols * bits
    if pad:
        b = np.concatenate([b, np.zeros((rows, pad), np.uint8)], axis=1)
    return np.packbits(b, axis=1, bitorder="little").reshape(-1)


def shard_rows(layer: QuantizedLayer, rank: int, world: int,
               align: int = 1) -> tuple[QuantizedLayer, int, int]:
    """Column-parallel shard: output rows [r0, r1)."""
    p, s = layer.packed, layer.sparse
    r0, r1 = split_range(layer.rows, world, rank, align)
    k = p.levels() * p.groups_per_row
    stride = p.row_stride()
    a, b = int(s.row_ptr[r0]), int(s.row_ptr[r1])
    packed = PackedDense(p.bits, r1 - r0, p.cols, np.asarray(p.luts)[r0 * k:r1 * k],
                         np.asarray(p.payload)[r0 * stride:r1 * stride], p.groups_per_row)
    sparse = CsrMatrix(r1 - r0, s.cols, (np.asarray(s.row_ptr[r0:r1 + 1]) - a).astype(np.uint32),
                       np.asarray(s.col_idx)[a:b], np.asarray(s.values)[a:b])
    return (QuantizedLayer(f"{layer.name}.r{rank}", r1 - r0, layer.cols, packed, sparse,
                           min(layer.hybrid_top_k, r1 - r0)), r0, r1)


def shard_cols(layer: QuantizedLayer, rank: int, world: int,
               align: int = 32) -> tuple[QuantizedLayer, int, int]:
    """Row-parallel shard: input columns [c0, c1) (align-column boundaries)."""
    p, s = layer.packed, layer.sparse
    if p.groups_per_row != 1:
        raise ValueError("row-parallel sharding implemented for channel-wise LUTs")
    c0, c1 = split_range(layer.cols, world, rank, align)
    idx = _unpack_rows(p)[:, c0:c1]
    packed = PackedDense(p.bits, p.rows, c1 - c0, np.asarray(p.luts),
                         _pack_rows(idx, p.bits), 1)
    rp = np.asarray(s.row_ptr, np.int64)
    ci = np.asarray(s.col_idx, np.int64)
    keep = (ci >= c0) & (ci < c1)
    rows_of = np.repeat(np.arange(layer.rows), np.diff(rp))
    new_rp = np.zeros(layer.rows + 1, np.int64)
    np.add.at(new_rp, rows_of[keep] + 1, 1)
    new_rp = np.cumsum(new_rp).astype(np.uint32)
    sparse = CsrMatrix(layer.rows, c1 - c0, new_rp, (ci[keep] - c0).astype(np.uint16),
                       np.asarray(s.values)[keep])
    return (QuantizedLayer(f"{layer.name}.c{rank}", layer.rows, c1 - c0, packed, sparse,
                           layer.hybrid_top_k), c0, c1)


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
    """The 7 shards (QuantizedLayer) of one decoder layer for `rank`."""
    out = []
    for name, q in zip(DECODER, layers):
        if world == 1:
            out.append(q)
        elif name in ROW_PARALLEL:
            out.append(shard_cols(q, rank, world, align)[0])
        else:
            out.append(shard_rows(q, rank, world, align)[0])
    return out


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
