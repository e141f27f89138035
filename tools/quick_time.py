"""Quick device timing of the fused kernel (dev tool, not the bench contract).

Rotates through enough distinct device layers that the working set exceeds
L2, times K back-to-back launches with CUDA events on the launching stream.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096,11008x4096,4096x11008")
    ap.add_argument("--bits", default="3,4")
    ap.add_argument("--sparsity", type=float, default=0.0045)
    ap.add_argument("--kernels", default="fused,lut")
    ap.add_argument("--reps", type=int, default=200)
    args = ap.parse_args()
    import torch
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer
    from oracle.oracle import make_layer, make_x, to_quantized_layer
    kid = {"fused": N.KERNEL_FUSED, "lut": N.KERNEL_LUT, "csr": N.KERNEL_CSR,
           "reference": N.KERNEL_REFERENCE}
    st = torch.cuda.current_stream().cuda_stream
    for bits in [int(b) for b in args.bits.split(",")]:
        for shp in args.shapes.split(","):
            rows, cols = map(int, shp.split("x"))
            t0 = time.time()
            L = make_layer(rows, cols, bits, args.sparsity, seed=1)
            q = to_quantized_layer(L)
            nbytes = L.payload.nbytes
            nl = max(2, int(np.ceil(600e6 / nbytes)))
            dls = [DeviceLayer(q) for _ in range(nl)]
            t1 = time.time()
            x = torch.from_numpy(make_x(cols).view(np.int16)).cuda()
            y = torch.empty(rows, dtype=torch.float32, device="cuda")
            info = dls[0].info()
            for kn in args.kernels.split(","):
                k = kid[kn]
                for i in range(10):
                    dls[i % nl].gemv(k, x.data_ptr(), N.F16, y.data_ptr(), N.F32, st)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for i in range(args.reps):
                    dls[i % nl].gemv(k, x.data_ptr(), N.F16, y.data_ptr(), N.F32, st)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / args.reps
                ab = info.algorithmic_bytes if kn == "fused" else int(
                    N.lib.dsq_bytes_touched_estimate(rows, cols, bits, 0, 0))
                if kn == "reference":
                    ab = rows * cols * 2 + rows * 2 + cols * 2
                print(f"{kn:9s} {rows}x{cols} b{bits} nnz {L.nnz}: {us:8.2f} us/layer  "
                      f"{ab / us / 1e3:8.1f} GB/s  (workers {info.workers}, ctas {info.ctas}, "
                      f"{nl} layers rotated, setup {t1 - t0:.1f}s)", flush=True)
            del dls


if __name__ == "__main__":
    main()
