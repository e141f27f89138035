"""Persistent stack of INDEPENDENT layers (no dependency waits): pure
streaming + dense throughput of the stack kernel (dev tool)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from oracle.oracle import make_layer, make_x, to_quantized_layer
    rows, cols, bits = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 3))]
    sp = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0045
    n = int(sys.argv[5]) if len(sys.argv) > 5 else 64
    L = make_layer(rows, cols, bits, sp, seed=5)
    q = to_quantized_layer(L)
    dls = [DeviceLayer(q) for _ in range(n)]
    x = torch.from_numpy(make_x(cols).view(np.int16)).cuda()
    ys = [torch.empty(rows, dtype=torch.int16, device="cuda") for _ in range(n)]
    st = DeviceStack(dls, [-1] * n, [x.data_ptr()] * n, [y.data_ptr() for y in ys], N.F16)
    s = torch.cuda.Stream()
    for _ in range(3):
        st.run(s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5):
        st.run(s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    ab = int(N.lib.dsq_bytes_touched_estimate(rows, cols, bits, 0, L.nnz)) * n
    print(f"{rows}x{cols} b{bits} sp{sp} x{n}: {ms*1e3/n:.2f} us/layer  {ab/ms/1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
