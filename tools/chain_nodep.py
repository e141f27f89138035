"""The bench's decoder-layer chain with and without its data dependencies
(dev tool): same layers, same order, same rotation; `nodep` makes every
GEMV read an external x, so the difference is the cost of the grid-wide
layer dependencies (signal -> acquire -> x staging) on the critical path."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import bench
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from oracle.oracle import make_x, to_quantized_layer
    host = bench.build_host_layers()
    qls = [to_quantized_layer(L, name=n) for L, (n, _, _) in zip(host, bench.SHAPES)]
    bytes_step = sum(int(N.lib.dsq_bytes_touched_estimate(r, c, 3, 0, L.nnz))
                     for L, (_, r, c) in zip(host, bench.SHAPES))
    rot, steps = 16, 50
    dls = [[DeviceLayer(q) for q in qls] for _ in range(rot)]
    xs = {c: torch.from_numpy(make_x(c).view(np.int16)).cuda() for c in (4096, 11008)}
    ys = [[torch.empty(r, dtype=torch.int16, device="cuda") for (_, r, _) in bench.SHAPES]
          for _ in range(rot)]
    for mode in ("dep", "nodep"):
        layers, deps, xp, yp = [], [], [], []
        prev = -1
        for s in range(steps):
            base = len(layers)
            for j, dl in enumerate(dls[s % rot]):
                layers.append(dl)
                c = bench.SHAPES[j][2]
                if mode == "nodep" or (bench.CHAIN_IN[j] < 0 and prev < 0):
                    deps.append(-1)
                    xp.append(xs[c].data_ptr())
                else:
                    deps.append(prev if bench.CHAIN_IN[j] < 0 else base + bench.CHAIN_IN[j])
                    xp.append(0)
                yp.append(ys[s % rot][j].data_ptr())
            prev = base + 6
        st = DeviceStack(layers, deps, xp, yp, N.F16)
        st.run(0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.run(0)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{mode:6s}: {ms * 1e3 / steps:.2f} us/step  {bytes_step * steps / ms / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
