"""GPU parity at the full BASELINE shapes (configs[0], [2], [3]) and of the hot
decode itself.

* The A fragments the hot kernels build (PRMT byte-plane decode, tile.cuh
  span3_frags / span4_frags) are dumped by dsq_cuda_dump_frags and must equal
  ref::dequant_dense (reference kernels.cpp:149-159) bit for bit.
* configs[0]: 4096 x 4096, 4-bit, dense-only, batch 1.
* configs[2] / [3] shapes (LLaMA-13B 5120 / 13824, LLaMA-65B 8192 / 22016),
  3-bit + 0.45% CSR: every single-layer product, and a 7-GEMV decoder chain
  (v, q, o, k, up, gate, down; the bench's dependency pattern) in one
  persistent launch with every layer checked on its actual device input.
* A served 13B decoder chain (16-consumer serving kernels) against regular
  runs of the same chain, step by step.

Tolerances (north_star): normwise max|dy| / max|y| <= 1e-3, and the
condition-aware max_r |dy_r| / sum_c |w_rc x_c| <= 5e-6 for fp32 outputs
(fp32 accumulation of exact fp16 products vs the reference's double).
"""
import numpy as np
import pytest

from oracle.oracle import Layer, make_layer, make_x, to_quantized_layer

pytestmark = pytest.mark.gpu

TOL_NORM = 1e-3
TOL_COND = 5e-6
DECODER = ["v", "q", "o", "k", "up", "gate", "down"]
CHAIN_IN = [-1, -1, 0, -1, 2, 2, 4]
MODELS = {"13b": (5120, 13824), "65b": (8192, 22016)}


def abs_scale(oracle, L: Layer, x32):
    """sum_c |w_rc x_c| through the oracle: the same layer with |LUT| and |delta|."""
    A = Layer(L.bits, L.rows, L.cols, L.assign, np.abs(L.luts16), L.payload, L.row_ptr,
              L.col_idx, np.abs(L.values16))
    return oracle.fused_dns_matvec(A, np.abs(x32), 0, nthreads=16)


def run_gemv(torch, dl, kernel, x16, y_f32=True):
    import paper_2306_07629_b200._native as N
    xt = torch.from_numpy(np.ascontiguousarray(x16).view(np.int16)).cuda()
    yt = torch.empty(dl.rows, dtype=torch.float32 if y_f32 else torch.float16, device="cuda")
    dl.gemv(kernel, xt.data_ptr(), N.F16, yt.data_ptr(), N.F32 if y_f32 else N.F16,
            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return yt.float().cpu().numpy().astype(np.float64)


def check(y, ref, scale, cond=True):
    d = np.abs(y - ref)
    norm = d.max() / max(np.abs(ref).max(), 1e-30)
    assert norm <= TOL_NORM, f"normwise {norm:.3e}"
    if cond:
        c = (d / np.maximum(scale, 1e-30)).max()
        assert c <= TOL_COND, f"condition-aware {c:.3e}"


@pytest.mark.parametrize("rows,cols,bits,skew", [
    (64, 256, 3, "uniform"), (33, 70, 3, "uniform"), (97, 300, 4, "halfrow"),
    (256, 1000, 4, "zipf"), (1, 33, 3, "uniform"),
    (4096, 4096, 4, "uniform"),      # configs[0]
    (11008, 4096, 3, "uniform"),     # configs[1] up / gate
    (5120, 13824, 3, "uniform"),     # configs[2] down
])
def test_hot_decode_fragments_bit_exact(torch, oracle, rows, cols, bits, skew):
    """The fp16 A fragments of the timed decode == ref::dequant_dense, bit for bit."""
    from paper_2306_07629_b200 import DeviceLayer
    L = make_layer(rows, cols, bits, 0.0045, seed=rows + 3 * cols + bits, skew=skew)
    dl = DeviceLayer(to_quantized_layer(L))
    w = torch.full((rows * cols,), -1, dtype=torch.int16, device="cuda")
    dl.dump_frags(w.data_ptr())
    torch.cuda.synchronize()
    got = w.cpu().numpy().view(np.float16)
    want = oracle.dequant_dense(L)  # f32 widening of the fp16 centroids (exact)
    assert np.array_equal(got.view(np.uint16), want.astype(np.float16).view(np.uint16))
    assert np.array_equal(got.astype(np.float32), want)


def test_config0_4bit_dense_full(torch, oracle):
    """BASELINE configs[0]: 4096 x 4096, 4-bit, no outliers, batch 1."""
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer
    L = make_layer(4096, 4096, 4, 0.0, seed=1234)
    assert L.nnz == 0
    x16 = make_x(4096, seed=99)
    x32 = x16.astype(np.float32)
    dl = DeviceLayer(to_quantized_layer(L))
    scale = abs_scale(oracle, L, x32)
    y = run_gemv(torch, dl, N.KERNEL_FUSED, x16)
    ref = oracle.fused_dns_matvec(L, x32, 10, nthreads=16)
    check(y, ref, scale)
    check(run_gemv(torch, dl, N.KERNEL_LUT, x16), oracle.lut_matvec(L, x32, nthreads=16), scale)
    assert np.array_equal(run_gemv(torch, dl, N.KERNEL_FUSED, x16), y)  # deterministic
    y2 = run_gemv(torch, dl, N.KERNEL_FUSED, (x32 * 2).astype(np.float16))
    assert np.array_equal(y2, 2 * y)  # exact power-of-two scaling


_CACHE = {}


def model_layers(name):
    """The three distinct shapes of a decoder layer (q/k/v/o, up/gate, down)."""
    if name not in _CACHE:
        h, f = MODELS[name]
        sq = make_layer(h, h, 3, 0.0045, seed=h + 1)
        up = make_layer(f, h, 3, 0.0045, seed=f + 2)
        dn = make_layer(h, f, 3, 0.0045, seed=h + f + 3, skew="zipf" if name == "13b" else
                        "uniform")
        _CACHE.clear()
        _CACHE[name] = {"sq": sq, "up": up, "down": dn}
    return _CACHE[name]


def decoder_layer_objects(name):
    Ls = model_layers(name)
    return [Ls["sq"], Ls["sq"], Ls["sq"], Ls["sq"], Ls["up"], Ls["up"], Ls["down"]]


@pytest.mark.parametrize("model,which", [(m, w) for m in ("13b", "65b")
                                          for w in ("sq", "up", "down")])
def test_full_size_13b_65b_single_layer(torch, oracle, model, which):
    """configs[2]/[3] shapes, 3-bit + 0.45% CSR, single-layer products."""
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer
    L = model_layers(model)[which]
    x16 = make_x(L.cols, seed=L.rows ^ L.cols)
    x32 = x16.astype(np.float32)
    dl = DeviceLayer(to_quantized_layer(L))
    scale = abs_scale(oracle, L, x32)
    y = run_gemv(torch, dl, N.KERNEL_FUSED, x16)
    check(y, oracle.fused_dns_matvec(L, x32, 10, nthreads=16), scale)
    check(run_gemv(torch, dl, N.KERNEL_LUT, x16), oracle.lut_matvec(L, x32, nthreads=16), scale)
    y16 = run_gemv(torch, dl, N.KERNEL_FUSED, x16, y_f32=False)
    assert np.array_equal(y16, y.astype(np.float16).astype(np.float64))


def test_4bit_16_consumer_single_layer(torch, oracle):
    """A 13B-shaped 4-bit layer: the plan picks the 16-consumer 4-bit kernel."""
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer
    L = make_layer(13824, 5120, 4, 0.0045, seed=4)
    x16 = make_x(5120, seed=8)
    x32 = x16.astype(np.float32)
    dl = DeviceLayer(to_quantized_layer(L))
    y = run_gemv(torch, dl, N.KERNEL_FUSED, x16)
    check(y, oracle.fused_dns_matvec(L, x32, 10, nthreads=16), abs_scale(oracle, L, x32))


def _chain(torch, name, steps, y_dtype_f16=True):
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    Ls = decoder_layer_objects(name)
    h = MODELS[name][0]
    uniq = {}
    dls = []
    for L in Ls:
        if id(L) not in uniq:
            uniq[id(L)] = DeviceLayer(to_quantized_layer(L))
        dls.append(uniq[id(L)])
    x16 = make_x(h, seed=5)
    xt = torch.from_numpy(x16.view(np.int16)).cuda()
    ys, layers, deps, xp = [], [], [], []
    prev_down = -1
    for s in range(steps):
        base = len(layers)
        for j, dl in enumerate(dls):
            layers.append(dl)
            ys.append(torch.zeros(dl.rows, dtype=torch.int16, device="cuda"))
            if CHAIN_IN[j] < 0:
                deps.append(prev_down)
                xp.append(xt.data_ptr() if prev_down < 0 else 0)
            else:
                deps.append(base + CHAIN_IN[j])
                xp.append(0)
        prev_down = base + len(dls) - 1
    st = DeviceStack(layers, deps, xp, [y.data_ptr() for y in ys], N.F16)
    return Ls * steps, deps, x16, ys, st


@pytest.mark.parametrize("model", ["13b", "65b"])
def test_full_size_decoder_chain(torch, oracle, model):
    """7-GEMV decoder chains (2 steps = 14 GEMVs) in one persistent launch:
    every output equals the oracle on that layer's actual device input."""
    Ls, deps, x16, ys, st = _chain(torch, model, 2)
    st.run(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    outs = [y.cpu().numpy().view(np.float16) for y in ys]
    for i, (L, d) in enumerate(zip(Ls, deps)):
        xin = (x16 if d < 0 else outs[d]).astype(np.float32)
        ref = oracle.fused_dns_matvec(L, xin, 10, nthreads=16)
        got = outs[i].astype(np.float64)
        # fp16 output: one rounding of the fp32 result (+ fp32 accumulation)
        tol = np.abs(ref).max() * 1e-3 + 1e-6
        assert np.abs(got - ref).max() <= tol, (i, DECODER[i % 7])
    st.run(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for y, o in zip(ys, outs):  # bit-identical reruns
        assert np.array_equal(y.cpu().numpy().view(np.float16), o)


def test_served_13b_decoder_chain_matches_regular_runs(torch, oracle):
    """The serving loop (16-consumer served kernel at 13B widths) over the
    bench's 7-GEMV launch order: gated layers v, q, k (gate = step), o between
    them, notify on down.  Each step's host output equals a regular run of the
    same chain on that step's x, and down's output matches the oracle."""
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    K = 3
    Ls = decoder_layer_objects("13b")
    h = MODELS["13b"][0]
    uniq = {}
    dls = []
    for L in Ls:
        if id(L) not in uniq:
            uniq[id(L)] = DeviceLayer(to_quantized_layer(L))
        dls.append(uniq[id(L)])
    x_dev = torch.zeros(h, dtype=torch.int16, device="cuda")
    outs = [[torch.zeros(dl.rows, dtype=torch.int16, device="cuda") for dl in dls]
            for _ in range(K)]
    layers, deps, xp, yp, gate, notify = [], [], [], [], [], []
    for k in range(K):
        base = len(layers)
        for j, dl in enumerate(dls):
            layers.append(dl)
            deps.append(-1 if CHAIN_IN[j] < 0 else base + CHAIN_IN[j])
            xp.append(x_dev.data_ptr() if CHAIN_IN[j] < 0 else 0)
            yp.append(outs[k][j].data_ptr())
            gate.append(k + 1 if CHAIN_IN[j] < 0 else 0)
            notify.append(k + 1 if j == 6 else 0)
    served = DeviceStack(layers, deps, xp, yp, N.F16, serve_gate=gate, serve_notify=notify)
    y_host = torch.zeros(h, dtype=torch.int16).pin_memory()
    x_pins = [torch.from_numpy(make_x(h, seed=300 + k).view(np.int16).copy()).pin_memory()
              for k in range(K)]
    s = torch.cuda.current_stream().cuda_stream
    torch.cuda.synchronize()
    served.serve_begin(x_dev.data_ptr(), h * 2, y_host.data_ptr(), h * 2, s)
    got = []
    for k in range(K):
        served.serve_step(x_pins[k].data_ptr())
        got.append(y_host.numpy().copy())
    served.serve_end()
    # regular runs of one step of the same chain
    ref_y = [torch.zeros(dl.rows, dtype=torch.int16, device="cuda") for dl in dls]
    reg = DeviceStack(dls, CHAIN_IN, [x_dev.data_ptr() if c < 0 else 0 for c in CHAIN_IN],
                      [y.data_ptr() for y in ref_y], N.F16)
    for k in range(K):
        x_dev.copy_(x_pins[k].cuda())
        reg.run(s)
        torch.cuda.synchronize()
        for j in range(7):
            assert np.array_equal(outs[k][j].cpu().numpy(), ref_y[j].cpu().numpy()), (k, j)
        assert np.array_equal(got[k], ref_y[6].cpu().numpy()), k
        up = ref_y[4].cpu().numpy().view(np.float16).astype(np.float32)
        want = oracle.fused_dns_matvec(Ls[6], up, 10, nthreads=16)
        g = got[k].view(np.float16).astype(np.float64)
        assert np.abs(g - want).max() <= np.abs(want).max() * 1e-3 + 1e-6, k
