"""Per-consumer-warp cycle breakdown of the persistent stack kernel (dev tool).

Runs n independent layers of one shape with DSQ_STACK_DBG=4 (the kernel's
clock64 profile) and prints, averaged over CTAs and consumer warps, the cycles
spent waiting for x / partial buffers, waiting for ring data, decoding, and in
the CSR phase, plus the kernel time."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

os.environ["DSQ_STACK_TRACE"] = "1"
os.environ["DSQ_STACK_DBG"] = str(4 | int(os.environ.get("DSQ_STACK_DBG_EXTRA", "0")))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from oracle.oracle import make_layer, make_x, to_quantized_layer
    rows, cols, bits = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 3))]
    sp = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0045
    n = int(sys.argv[5]) if len(sys.argv) > 5 else 32
    L = make_layer(rows, cols, bits, sp, seed=5)
    q = to_quantized_layer(L)
    dls = [DeviceLayer(q) for _ in range(n)]
    x = torch.from_numpy(make_x(cols).view(np.int16)).cuda()
    ys = [torch.empty(rows, dtype=torch.int16, device="cuda") for _ in range(n)]
    st = DeviceStack(dls, [-1] * n, [x.data_ptr()] * n, [y.data_ptr() for y in ys], N.F16)
    for _ in range(2):
        st.run(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.run(0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    G = torch.cuda.get_device_properties(0).multi_processor_count
    NC = int(os.environ.get("DSQ_STACK_CONSUMERS", "16"))
    lib = N.lib
    lib.dsq_cuda_stack_trace.restype = C.c_uint64
    lib.dsq_cuda_stack_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
    buf = np.zeros(max(G * n * 12, G * 24 * 5), np.int64)
    got = lib.dsq_cuda_stack_trace(st.handle, buf.ctypes.data, buf.size)
    assert got, "trace buffer missing"
    prof = buf[: G * NC * 5].reshape(G, NC, 5).astype(np.float64)
    names = ["x/part wait", "ring wait", "chunk/segment bookkeeping", "unit loops", "layer top"]
    tot = prof.sum(axis=2).mean()
    print(f"{rows}x{cols} b{bits} sp{sp} x{n}: {ms * 1e3 / n:.2f} us/layer; consumer cycles/layer "
          f"(mean over CTAs, warps): " + ", ".join(
              f"{nm} {prof[:, :, k].mean() / n:.0f} ({prof[:, :, k].mean() / tot * 100:.0f}%)"
              for k, nm in enumerate(names)))
    w = (prof[:, :, 2] + prof[:, :, 3]).mean(axis=0) / n
    print("  dense (bookkeeping + loops) cycles/layer per warp:", " ".join(f"{v:.0f}" for v in w))


if __name__ == "__main__":
    main()
