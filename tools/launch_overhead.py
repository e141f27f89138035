"""Fixed cost of an isolated persistent-kernel launch (dev tool): 200
single-layer fused products (K7, one launch each) of a small, a medium and a
4096^2 3-bit layer, back to back in one captured CUDA graph, rotating over 8
device copies; prints microseconds per launch (3.46 us
for 128x256).

usage: python tools/launch_overhead.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_07629_b200._native as N
from paper_2306_07629_b200 import DeviceLayer
from oracle.oracle import make_layer, make_x, to_quantized_layer
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for (r, c) in [(128, 256), (1024, 1024), (4096, 4096)]:
    L = make_layer(r, c, 3, 0.0045, seed=1)
    dls = [DeviceLayer(to_quantized_layer(L)) for _ in range(8)]
    x = torch.from_numpy(make_x(c).view(np.int16)).cuda()
    y = torch.empty(r, dtype=torch.int16, device='cuda')
    def run(k):
        for i in range(k): dls[i % 8].gemv(N.KERNEL_FUSED, x.data_ptr(), N.F16, y.data_ptr(), N.F16, st.cuda_stream)
    run(16); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st): run(200)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(r, c, 'isolated us per launch', e0.elapsed_time(e1) * 1e3 / 200)
