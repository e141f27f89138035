"""Timeline of the serving loop (dev tool): a served 7B decoder-layer stack
with DSQ_STACK_TRACE=1, fed step by step; prints per step the GPU-side
compute span (first gated layer's x issued -> last layer signalled) and the
gap to the next step's x (host round trip + PCIe copy), in microseconds."""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ["DSQ_STACK_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
SLOTS = ["ld_start", "csr_staged", "dep_met", "x_issued", "c_start", "x_ready", "dense_done",
         "csr_done", "signaled", "prod_first", "all_dense", "final_done"]


def main():
    import torch
    import bench
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from oracle.oracle import make_x, to_quantized_layer
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    host = bench.build_host_layers()
    qls = [to_quantized_layer(L, name=n) for L, (n, _, _) in zip(host, bench.SHAPES)]
    rot = 4
    dls = [[DeviceLayer(q) for q in qls] for _ in range(rot)]
    x_dev = torch.zeros(4096, dtype=torch.int16, device="cuda")
    ys = [[torch.empty(r, dtype=torch.int16, device="cuda") for (_, r, _) in bench.SHAPES]
          for _ in range(rot)]
    y_host = torch.zeros(4096, dtype=torch.int16).pin_memory()
    x_host = torch.from_numpy(make_x(4096, seed=7).view(np.int16)).pin_memory()
    layers, deps, xp, yp, gate, notify = [], [], [], [], [], []
    for k in range(K):
        slot, base = k % rot, len(layers)
        for j, dl in enumerate(dls[slot]):
            last = j == 6
            layers.append(dl)
            deps.append(-1 if bench.CHAIN_IN[j] < 0 else base + bench.CHAIN_IN[j])
            xp.append(x_dev.data_ptr() if bench.CHAIN_IN[j] < 0 else 0)
            gate.append(k + 1 if bench.CHAIN_IN[j] < 0 else 0)
            yp.append(ys[slot][j].data_ptr())
            notify.append(k + 1 if last else 0)
    st = DeviceStack(layers, deps, xp, yp, N.F16, serve_gate=gate, serve_notify=notify)
    torch.cuda.synchronize()
    host_us = []
    for rep in range(2):
        st.serve_begin(x_dev.data_ptr(), 8192, y_host.data_ptr(), 8192, 0)
        for k in range(K):
            t0 = time.perf_counter()
            st.serve_step(x_host.data_ptr())
            host_us.append((time.perf_counter() - t0) * 1e6)
        st.serve_end()
    lib = N.lib
    lib.dsq_cuda_stack_trace.restype = C.c_uint64
    lib.dsq_cuda_stack_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
    n = len(layers)
    G = torch.cuda.get_device_properties(0).multi_processor_count
    buf = np.zeros(max(G * n * len(SLOTS), G * 24 * 5), np.uint64)
    got = lib.dsq_cuda_stack_trace(st.handle, buf.ctypes.data, buf.size)
    assert got == buf.size, got
    t = buf[: G * n * len(SLOTS)].reshape(G, n, len(SLOTS)).astype(np.float64)
    t0 = t[t > 0].min()
    t = np.where(t > 0, (t - t0) / 1e3, np.nan)
    gated = [j for j in range(7) if bench.CHAIN_IN[j] < 0]
    XI, XR, SIG = SLOTS.index("x_issued"), SLOTS.index("x_ready"), SLOTS.index("signaled")
    print("host us per serve_step (2nd pass):", np.round(host_us[K:], 1).tolist())
    prev = None
    for k in range(K):
        q = 7 * k + gated[0]
        xi = np.nanmin(t[:, q, XI])
        xr = np.nanmedian(t[:, q, XR])
        done = np.nanmax(t[:, 7 * k + 6, SIG])
        per = [np.nanmax(t[:, 7 * k + j, SIG]) for j in range(7)]
        print(f"step {k}: x issued {xi:9.1f}  x ready(med) {xr - xi:5.1f}  compute {done - xi:6.1f}"
              + (f"  gap from prev done {xi - prev:6.1f}" if prev is not None else "")
              + "  layer ends " + " ".join(f"{v - xi:5.1f}" for v in per))
        prev = done


if __name__ == "__main__":
    main()
