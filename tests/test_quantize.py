"""GPU channel-wise quantization (K9, csrc/quantize.cu) against the UNMODIFIED
reference dsq::quantize_channelwise (src/nuq.cpp:673-779) compiled in
oracle/_ref: codebooks, assignments and both objectives must be identical
(bit for bit) -- weighted / unweighted k-means and round-to-nearest,
channel-wise and grouped, with masks, zero sensitivities (uniform-weight
fallback), rows with at most 2^bits distinct values, duplicated values and
ties.  The CPU tests check the argument validation against the reference."""
import numpy as np
import pytest

from paper_2306_07629_b200 import _native as N
from paper_2306_07629_b200.quantize import QuantConfig, quantize_channelwise

METHOD = {"weighted_kmeans": 0, "unweighted_kmeans": 1, "rtn": 2}


def _case(rows, cols, seed, kind="normal"):
    rng = np.random.default_rng(seed)
    w = rng.standard_t(4, size=(rows, cols)).astype(np.float32) * np.float32(0.02)
    sens = (rng.normal(size=(rows, cols)) ** 2).astype(np.float32)
    if kind == "ties":  # coarse grid: many duplicated values and equal-cost cuts
        w = (np.round(w / 0.01) * 0.01).astype(np.float32)
    if kind == "zero_sens":
        sens[:] = 0
    if kind == "sparse_sens":
        sens[rng.random(sens.shape) < 0.7] = 0
    if kind == "few_distinct":
        w = rng.choice(np.array([-0.5, 0.0, 0.25, 1.0], np.float32), size=(rows, cols))
    return w, sens


def _check(reference, w, sens, bits, group_size=0, mask=None, method="weighted_kmeans",
           max_iters=100, tol=1e-6):
    rc, cent, assign, obj, mse = reference.quantize_channelwise(
        w, sens, bits, group_size, max_iters, tol, mask, METHOD[method])
    assert rc == 0, reference.err()
    res = quantize_channelwise(w, sens, QuantConfig(bits=bits, group_size=group_size,
                                                    kmeans_max_iters=max_iters, kmeans_tol=tol),
                               mask=mask, method=method)
    np.testing.assert_array_equal(res.codebooks.view(np.uint32), cent.view(np.uint32))
    np.testing.assert_array_equal(res.assignment, assign)
    assert res.weighted_objective == obj and res.unweighted_mse_sum == mse
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("kind", ["normal", "ties", "zero_sens", "sparse_sens", "few_distinct"])
def test_weighted_kmeans_matches_reference(torch, reference, bits, kind):
    w, sens = _case(12, 384, seed=bits * 10 + len(kind), kind=kind)
    _check(reference, w, sens, bits)


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["unweighted_kmeans", "rtn"])
def test_other_methods_match_reference(torch, reference, method):
    w, sens = _case(10, 256, seed=7)
    _check(reference, w, sens, 3, method=method)


@pytest.mark.gpu
def test_grouped_and_masked_match_reference(torch, reference):
    w, sens = _case(8, 512, seed=3)
    rng = np.random.default_rng(4)
    mask = (rng.random(w.shape) < 0.01).astype(np.uint8)
    res = _check(reference, w, sens, 3, group_size=128, mask=mask)
    assert res.groups_per_row == 4
    assert (res.assignment[mask.astype(bool)] == 0xFFFF).all()
    _check(reference, w, sens, 4, mask=mask)


@pytest.mark.gpu
def test_short_budget_and_loose_tolerance(torch, reference):
    w, sens = _case(6, 300, seed=9)
    _check(reference, w, sens, 3, max_iters=2)
    _check(reference, w, sens, 3, tol=1e-2)


@pytest.mark.gpu
def test_llama_row_length(torch, reference):
    """rows of LLaMA-7B length (4096 columns), the pipeline's 3-bit setting."""
    w, sens = _case(8, 4096, seed=11)
    _check(reference, w, sens, 3)


@pytest.mark.gpu
def test_empty_channel_error(torch, reference):
    w, sens = _case(4, 64, seed=1)
    mask = np.zeros(w.shape, np.uint8)
    mask[2] = 1
    rc = reference.quantize_channelwise(w, sens, 3, 0, 100, 1e-6, mask, 0)[0]
    with pytest.raises(N.DsqError) as e:
        quantize_channelwise(w, sens, QuantConfig(bits=3), mask=mask)
    assert e.value.code == rc == 13  # errc::empty_channel


@pytest.mark.parametrize("case", ["bits", "iters", "tol", "group", "frac", "nonfinite", "empty"])
def test_validation_matches_reference(reference, case):
    """Argument checks run before any device work (CPU)."""
    w, sens = _case(4, 64, seed=2)
    cfg = dict(bits=3, group_size=0, max_iters=100, tol=1e-6)
    qc = QuantConfig(bits=3)
    if case == "bits":
        cfg["bits"], qc.bits = 9, 9
    elif case == "iters":
        cfg["max_iters"], qc.kmeans_max_iters = 0, 0
    elif case == "tol":
        cfg["tol"], qc.kmeans_tol = -1.0, -1.0
    elif case == "group":
        cfg["group_size"], qc.group_size = 48, 48
    elif case == "frac":
        qc.outlier_fraction = 0.2
    elif case == "nonfinite":
        w[1, 3] = np.inf
    elif case == "empty":
        w, sens = np.zeros((0, 64), np.float32), np.zeros((0, 64), np.float32)
    with pytest.raises(N.DsqError) as e:
        quantize_channelwise(w, sens, qc)
    if case == "frac":  # the shim takes the default fractions; the rule is QuantConfig's
        assert e.value.code == 11
        return
    if case == "empty":
        assert e.value.code == 4  # errc::empty_dimension (WeightMatrix::validate)
        return
    rc = reference.quantize_channelwise(w, sens, cfg["bits"], cfg["group_size"],
                                        cfg["max_iters"], cfg["tol"])[0]
    assert e.value.code == rc != 0


# ---- the whole quantize_layer pipeline (decompose K10 + k-means K9 + pack) ----

def _ref_layer_arrays(reference, w, sens, bits, sf, of, top_k=10):
    rl = reference.quantize(w, sens, w.shape[0], w.shape[1], bits, sf, of, top_k)
    a = rl.arrays()
    return (a["luts"], a["payload"], a["row_ptr"], a["col_idx"], a["values"]), \
        float(reference.lib.ref_avg_bits(rl.h))


@pytest.mark.gpu
@pytest.mark.parametrize("bits,sf,of,kind", [
    (3, 0.0005, 0.004, "normal"),       # the pipeline defaults (0.45%)
    (4, 0.0005, 0.004, "normal"),
    (3, 0.01, 0.02, "ties"),            # equal magnitudes: index tie-break
    (3, 0.02, 0.01, "zero_sens"),       # all-zero sensitivity: index tie-break
    (2, 0.0, 0.05, "sparse_sens"),
    (3, 0.05, 0.0, "normal"),
])
def test_quantize_layer_matches_reference(torch, reference, bits, sf, of, kind):
    from paper_2306_07629_b200.quantize import quantize_layer
    w, sens = _case(16, 512, seed=bits + int(1000 * sf), kind=kind)
    (luts, payload, row_ptr, col_idx, values), avg = _ref_layer_arrays(
        reference, w, sens, bits, sf, of)
    layer, stats = quantize_layer(w, sens, QuantConfig(bits=bits, sensitive_fraction=sf,
                                                       outlier_fraction=of))
    np.testing.assert_array_equal(np.asarray(layer.packed.luts, np.float32).view(np.uint32),
                                  luts.view(np.uint32))
    np.testing.assert_array_equal(np.asarray(layer.packed.payload, np.uint8), payload)
    nnz = int(row_ptr[-1])
    np.testing.assert_array_equal(np.asarray(layer.sparse.row_ptr, np.uint32), row_ptr)
    np.testing.assert_array_equal(np.asarray(layer.sparse.col_idx, np.uint16), col_idx[:nnz])
    np.testing.assert_array_equal(np.asarray(layer.sparse.values, np.float32).view(np.uint32),
                                  values[:nnz].view(np.uint32))
    assert stats["avg_bits"] == avg
    assert stats["sensitive_count"] + stats["outlier_count"] == nnz


@pytest.mark.gpu
def test_quantize_layer_llama_shape_and_device_product(torch, reference, oracle):
    """A 4096-column layer quantized on the GPU equals the reference's and
    runs through the hot path (the fused product against the oracle)."""
    from oracle.oracle import make_x
    from paper_2306_07629_b200 import fused_dns_matvec
    from paper_2306_07629_b200.quantize import quantize_layer
    w, sens = _case(64, 4096, seed=5)
    (luts, payload, row_ptr, *_), _ = _ref_layer_arrays(reference, w, sens, 3, 0.0005, 0.004)
    layer, _ = quantize_layer(w, sens, QuantConfig(bits=3))
    assert np.array_equal(np.asarray(layer.packed.payload, np.uint8), payload)
    assert np.array_equal(np.asarray(layer.packed.luts, np.float32), luts)
    x = make_x(4096, seed=1).astype(np.float32)
    y = fused_dns_matvec(layer, x)
    ref = reference.quantize(w, sens, 64, 4096, 3, 0.0005, 0.004).matvec("fused", x)
    assert np.abs(y - ref).max() <= np.abs(ref).max() * 1e-3


@pytest.mark.parametrize("case", ["overflow", "wide"])
def test_decompose_validation(case):
    from paper_2306_07629_b200.quantize import decompose
    if case == "overflow":  # ceil(0.05*4)+ceil(0.05*4) = 2 < 4 ok; 2x2 -> 1+1 < 4; 1x1 -> 2 >= 1
        w, s = np.ones((1, 1), np.float32), np.ones((1, 1), np.float32)
        code = 12  # errc::fraction_overflow
        cfg = QuantConfig(sensitive_fraction=0.05, outlier_fraction=0.05)
    else:
        w, s = np.ones((1, 65536), np.float32), np.ones((1, 65536), np.float32)
        code = 5  # errc::dimension_overflow
        cfg = QuantConfig()
    with pytest.raises(N.DsqError) as e:
        decompose(w, s, cfg)
    assert e.value.code == code
