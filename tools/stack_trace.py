"""Timeline of the persistent stack kernel (dev tool).

Builds the bench workload (LLaMA-7B decoder-layer chain), runs a short stack
with DSQ_STACK_TRACE=1 and prints, per layer, the median/max over CTAs of each
milestone relative to the kernel's first timestamp (microseconds)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

os.environ["DSQ_STACK_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
SLOTS = ["ld_start", "csr_staged", "dep_met", "x_issued", "c_start", "x_ready", "dense_done",
         "csr_done", "signaled", "prod_first", "all_dense", "final_done"]
SHOW = ["dep_met", "x_issued", "c_start", "x_ready", "dense_done", "csr_staged", "csr_done",
        "all_dense", "final_done", "signaled"]


def main():
    import torch
    import bench
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from oracle.oracle import make_x, to_quantized_layer
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    if len(sys.argv) > 2:  # independent layers of one shape: rows cols [n]
        return indep(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 24)
    host = bench.build_host_layers()
    qls = [to_quantized_layer(L, name=n) for L, (n, _, _) in zip(host, bench.SHAPES)]
    rot = 4
    dls = [[DeviceLayer(q) for q in qls] for _ in range(rot)]
    xs = [torch.from_numpy(make_x(4096, seed=i).view(np.int16)).cuda() for i in range(rot)]
    ys = [[torch.empty(r, dtype=torch.int16, device="cuda") for (_, r, _) in bench.SHAPES]
          for _ in range(rot)]
    layers, deps, xp, yp = [], [], [], []
    prev_down = -1
    for s in range(steps):
        slot = s % rot
        base = len(layers)
        for j, dl in enumerate(dls[slot]):
            layers.append(dl)
            if bench.CHAIN_IN[j] < 0 and prev_down < 0:
                deps.append(-1)
                xp.append(xs[slot].data_ptr())
            else:
                deps.append(prev_down if bench.CHAIN_IN[j] < 0 else base + bench.CHAIN_IN[j])
                xp.append(0)
            yp.append(ys[slot][j].data_ptr())
        prev_down = base + 6
    st = DeviceStack(layers, deps, xp, yp, N.F16)
    for _ in range(3):
        st.run(0)
    torch.cuda.synchronize()
    lib = N.lib
    lib.dsq_cuda_stack_trace.restype = C.c_uint64
    lib.dsq_cuda_stack_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
    n = len(layers)
    G = torch.cuda.get_device_properties(0).multi_processor_count
    buf = np.zeros(G * n * len(SLOTS), np.uint64)
    got = lib.dsq_cuda_stack_trace(st.handle, buf.ctypes.data, buf.size)
    assert got == buf.size, got
    t = buf.reshape(G, n, len(SLOTS)).astype(np.float64)
    t0 = t[t > 0].min()
    t = np.where(t > 0, (t - t0) / 1e3, np.nan)
    print(f"{'layer':>5} {'shape':>11} " + " ".join(f"{s:>14}" for s in SHOW))
    for l in range(n):
        name, r, c = bench.SHAPES[l % 7]
        cells = []
        for k in [SLOTS.index(s) for s in SHOW]:
            col = t[:, l, k]
            cells.append(f"{np.nanmedian(col):6.2f}/{np.nanmax(col):6.2f}")
        print(f"{l:5d} {name:>4}{r:>5}x{c:<5} " + " ".join(f"{c:>14}" for c in cells))
    tot = np.nanmax(t)
    mb = sum(int(N.lib.dsq_bytes_touched_estimate(r, c, 3, 0, L.nnz))
             for L, (_, r, c) in zip(host, bench.SHAPES)) * steps / 1e6
    print(f"kernel span {tot:.2f} us for {mb:.1f} MB -> {mb / tot * 1e3:.1f} GB/s")


def indep(rows, cols, n):
    import torch
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from oracle.oracle import make_layer, make_x, to_quantized_layer
    q = to_quantized_layer(make_layer(rows, cols, 3, 0.0045, seed=5))
    dls = [DeviceLayer(q) for _ in range(n)]
    x = torch.from_numpy(make_x(cols).view(np.int16)).cuda()
    ys = [torch.empty(rows, dtype=torch.int16, device="cuda") for _ in range(n)]
    st = DeviceStack(dls, [-1] * n, [x.data_ptr()] * n, [y.data_ptr() for y in ys], N.F16)
    for _ in range(3):
        st.run(0)
    torch.cuda.synchronize()
    lib = N.lib
    lib.dsq_cuda_stack_trace.restype = C.c_uint64
    lib.dsq_cuda_stack_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
    G = torch.cuda.get_device_properties(0).multi_processor_count
    buf = np.zeros(max(G * n * len(SLOTS), G * 24 * 5), np.uint64)
    assert lib.dsq_cuda_stack_trace(st.handle, buf.ctypes.data, buf.size)
    t = buf[: G * n * len(SLOTS)].reshape(G, n, len(SLOTS)).astype(np.float64)
    t0 = t[t > 0].min()
    t = np.where(t > 0, (t - t0) / 1e3, np.nan)
    print(f"{'layer':>5} " + " ".join(f"{s:>14}" for s in SHOW))
    for l in range(n):
        cells = [f"{np.nanmedian(t[:, l, k]):6.2f}/{np.nanmax(t[:, l, k]):6.2f}"
                 for k in [SLOTS.index(s) for s in SHOW]]
        print(f"{l:5d} " + " ".join(f"{c:>14}" for c in cells))


if __name__ == "__main__":
    main()
