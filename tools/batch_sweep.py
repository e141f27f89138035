"""Batch sweep (BASELINE configs[4]): LLaMA-7B layer shapes, batch 1/2/4/8/16,
3- and 4-bit, sparsity 0 / 0.05% / 0.45%, fused Dense-and-Sparse products.

Batch 1 runs the persistent tensor-core LUT-GEMV (K7, dsq_cuda_gemv batch=1);
batch 2..4 the same kernel with 2/4 x vectors sharing every decoded fragment
(when they fit in shared memory next to the ring), batch 5..16 (and the rest)
the batched LUT-GEMM K11 (csrc/bstream.cu: dense 16-row HMMA fragments, batch
in the N dimension, per-warp TMA rings, decode amortised over the batch).  Each configuration rotates
over enough distinct device layers that the working set exceeds L2 and
times back-to-back products with CUDA events.  Prints one JSON line per
(shape, bits, sparsity, batch): µs per product, weight-stream GB/s
(reference-charged bytes incl. B x/y vectors), TFLOP/s (2*B*(rows*cols+nnz)),
and the speed-up of the batch over B sequential batch-1 products.

usage: python tools/batch_sweep.py [--shapes 4096x4096,11008x4096,4096x11008]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096,11008x4096,4096x11008")
    ap.add_argument("--bits", default="3,4")
    ap.add_argument("--sparsity", default="0,0.0005,0.0045")
    ap.add_argument("--batches", default="1,2,4,8,16")
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    import torch
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer
    from oracle.oracle import make_layer, make_x, to_quantized_layer
    st = torch.cuda.current_stream().cuda_stream
    batches = [int(b) for b in args.batches.split(",")]
    for shp in args.shapes.split(","):
        rows, cols = map(int, shp.split("x"))
        for bits in [int(b) for b in args.bits.split(",")]:
            for sp in [float(s) for s in args.sparsity.split(",")]:
                L = make_layer(rows, cols, bits, sp, seed=3)
                q = to_quantized_layer(L)
                nl = max(2, int(np.ceil(400e6 / L.payload.nbytes)))
                dls = [DeviceLayer(q) for _ in range(nl)]
                base_us = None
                for B in batches:
                    x = torch.from_numpy(np.stack([make_x(cols, seed=b) for b in range(B)])
                                         .view(np.int16)).cuda()
                    y = torch.empty(B, rows, dtype=torch.float16, device="cuda")
                    for i in range(max(5, nl)):  # every rotated layer once (lazy scratch)
                        N.check(N.lib.dsq_cuda_gemv(dls[i % nl].handle, N.KERNEL_FUSED,
                                                    x.data_ptr(), N.F16, y.data_ptr(), N.F16,
                                                    B, st))
                    torch.cuda.synchronize()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for i in range(args.reps):
                        N.check(N.lib.dsq_cuda_gemv(dls[i % nl].handle, N.KERNEL_FUSED,
                                                    x.data_ptr(), N.F16, y.data_ptr(), N.F16,
                                                    B, st))
                    e1.record()
                    torch.cuda.synchronize()
                    us = e0.elapsed_time(e1) * 1e3 / args.reps
                    wbytes = int(N.lib.dsq_bytes_touched_estimate(rows, cols, bits, 0, L.nnz))
                    bytes_b = wbytes + (B - 1) * (rows + cols) * 2
                    flops = 2.0 * B * (rows * cols + L.nnz)
                    if B == 1:
                        base_us = us
                    print(json.dumps({
                        "shape": shp, "bits": bits, "sparsity": sp, "batch": B,
                        "kernel": ("K7 persistent (batch 1)" if B == 1 else
                                   f"K7 persistent NB={2 if B == 2 else 4} "
                                   "(K11 when the x vectors do not fit)" if B <= 4 else
                                   "K11 batched HMMA (TMA rings) + finish"),
                        "us": round(us, 3), "GBs": round(bytes_b / us / 1e3, 1),
                        "TFLOPs": round(flops / us / 1e6, 2),
                        "speedup_vs_B_x_batch1": round(B * base_us / us, 2) if base_us else None,
                        "layers_rotated": nl}), flush=True)
                del dls


if __name__ == "__main__":
    main()
