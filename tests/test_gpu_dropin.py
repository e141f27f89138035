"""The reference's free functions through the Python mirror (the same C ABI the
C++ drop-ins in include/dsq_cuda.hpp call): dense_matvec (kernels.hpp:35),
dequantize_layer (pipeline.cpp:49-75), bench_matvec (kernels.cpp:214-282),
lut_matvec / csr_matvec on bare PackedDense / CsrMatrix."""
import numpy as np
import pytest

from oracle.oracle import make_layer, make_x, to_quantized_layer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,cols", [(1, 1), (33, 70), (256, 1000), (4096, 4096)])
def test_dense_matvec_vs_oracle(torch, oracle, rows, cols):
    from paper_2306_07629_b200 import dense_matvec
    rng = np.random.default_rng(rows + cols)
    m = rng.standard_normal(rows * cols).astype(np.float32)
    x = rng.standard_normal(cols).astype(np.float32)
    y = dense_matvec(m, rows, cols, x)
    ref = oracle.dense_matvec(m, rows, cols, x)
    # fp64 accumulation of exact fp32 products in another order: ~1 ulp of double
    assert np.abs(y - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("rows,cols,bits,sp", [(64, 256, 3, 0.0045), (33, 70, 4, 0.02),
                                               (40, 128, 2, 0.01), (97, 300, 5, 0.05),
                                               (1024, 4096, 3, 0.0045)])
def test_dequantize_layer_bit_exact_vs_reference(torch, reference, rows, cols, bits, sp):
    from paper_2306_07629_b200 import dequantize_layer
    L = make_layer(rows, cols, bits, sp, seed=rows * cols + bits, skew="zipf")
    got = dequantize_layer(to_quantized_layer(L))
    want = np.zeros(rows * cols, np.float32)
    import ctypes as C
    rl = reference.layer(L)
    assert reference.lib.ref_dequantize_layer(rl.h, C.c_void_p(want.ctypes.data)) == 0
    assert np.array_equal(got.reshape(-1).view(np.uint32), want.view(np.uint32))


def test_bench_matvec_record(torch, reference):
    from paper_2306_07629_b200 import BenchKernel, bench_matvec
    L = make_layer(512, 1024, 3, 0.0045, seed=3)
    q = to_quantized_layer(L)
    x = make_x(1024).astype(np.float32)
    rl = reference.layer(L)
    for k, name in [(BenchKernel.lut, "lut"), (BenchKernel.csr, "csr"),
                    (BenchKernel.fused, "fused"), (BenchKernel.reference, "reference")]:
        rec = bench_matvec(q, x, 3, k)
        _, ref_bytes = rl.bench(name, x, 3)
        assert rec.repeats == 3 and len(rec.all_seconds) == 3 and rec.median_seconds > 0
        assert rec.bytes_touched == ref_bytes, name


def test_bare_packed_and_csr_products(torch, oracle):
    from paper_2306_07629_b200 import csr_matvec, lut_matvec
    L = make_layer(300, 1000, 3, 0.02, seed=8, skew="halfrow")
    q = to_quantized_layer(L)
    x = make_x(1000, seed=1).astype(np.float32)
    ref = oracle.lut_matvec(L, x)
    assert np.abs(lut_matvec(q.packed, x) - ref).max() <= 1e-5 * np.abs(ref).max()
    ref = oracle.csr_matvec(L, x)
    assert np.abs(csr_matvec(q.sparse, x) - ref).max() <= 1e-5 * np.abs(ref).max()


@pytest.mark.parametrize("rows,cols,bits,groups,sp", [(64, 256, 3, 4, 0.0045), (33, 96, 4, 2, 0.02),
                                                      (40, 128, 2, 8, 0.01), (17, 120, 5, 3, 0.05),
                                                      (512, 4096, 3, 32, 0.0045)])
def test_grouped_luts_on_device(torch, oracle, reference, rows, cols, bits, groups, sp):
    """Grouped LUTs (groups_per_row > 1, the grouping ablation,
    packfmt.hpp:28-31 / kernels.cpp:21-30) through the device products:
    unpack / dequant bit-exact, products within the fp32-accumulation
    tolerance, dequantize_layer bit-exact against the reference."""
    import ctypes as C
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, dequantize_layer, fused_dns_matvec, lut_matvec
    L = make_layer(rows, cols, bits, sp, seed=rows + groups * 7 + bits, skew="zipf", groups=groups)
    q = to_quantized_layer(L)
    dl = DeviceLayer(q)
    assert dl.info().groups_per_row == groups
    a = torch.empty(rows * cols, dtype=torch.int16, device="cuda")
    dl.unpack(a.data_ptr())
    w = torch.empty(rows * cols, dtype=torch.float32, device="cuda")
    dl.dequant(w.data_ptr(), 0)
    torch.cuda.synchronize()
    rc, assign = oracle.unpack(L.payload, bits, rows, cols)
    assert rc == 0 and np.array_equal(a.cpu().numpy().view(np.uint16), assign)
    assert np.array_equal(w.cpu().numpy(), oracle.dequant_dense(L))
    x = make_x(cols, seed=5).astype(np.float32)
    ref = oracle.fused_dns_matvec(L, x, 10)
    y = fused_dns_matvec(q, x)
    assert np.abs(y - ref).max() <= 1e-5 * max(np.abs(ref).max(), 1e-30)
    refl = oracle.lut_matvec(L, x)
    assert np.abs(lut_matvec(q.packed, x) - refl).max() <= 1e-5 * max(np.abs(refl).max(), 1e-30)
    # device products on device buffers, fp16 x / fp32 y
    xt = torch.from_numpy(x.astype(np.float16).view(np.int16)).cuda()
    yt = torch.empty(rows, dtype=torch.float32, device="cuda")
    dl.gemv(N.KERNEL_FUSED, xt.data_ptr(), N.F16, yt.data_ptr(), N.F32)
    torch.cuda.synchronize()
    assert np.abs(yt.cpu().numpy() - ref).max() <= 1e-5 * max(np.abs(ref).max(), 1e-30)
    want = np.zeros(rows * cols, np.float32)
    rl = reference.layer(L)
    assert reference.lib.ref_dequantize_layer(rl.h, C.c_void_p(want.ctypes.data)) == 0
    assert np.array_equal(dequantize_layer(q).reshape(-1).view(np.uint32), want.view(np.uint32))
