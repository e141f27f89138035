"""The product library without a GPU: it loads, exports every symbol the C
header declares, and its host-side validation mirrors the reference's error
taxonomy (no compute calls).  On a GPU-less box a valid layer fails loudly
with DSQ_E_NO_DEVICE -- there is no CPU fallback."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import make_layer, to_quantized_layer

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dsq_cuda.h"


def declared_symbols():
    txt = HEADER.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dsq_(?:cuda_)?\w+)\s*\(", txt)))


def test_library_loads_and_exports_header_symbols():
    import paper_2306_07629_b200._native as N
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(N.lib, s), f"missing export {s}"
        assert s in N.PROTOTYPES, f"no ctypes prototype for {s}"
    assert N.lib.dsq_cuda_abi_version() == 1


def test_bytes_touched_matches_oracle(oracle):
    import paper_2306_07629_b200._native as N
    rng = np.random.default_rng(1)
    for _ in range(200):
        r, c = int(rng.integers(1, 30000)), int(rng.integers(1, 65535))
        b, nnz = int(rng.integers(1, 9)), int(rng.integers(0, 10 ** 6))
        assert N.lib.dsq_bytes_touched_estimate(r, c, b, 0, nnz) == oracle.bytes_touched(
            r, c, b, 0, nnz)


def _create(layer):
    from paper_2306_07629_b200 import DeviceLayer
    return DeviceLayer(layer)


def _errc(layer):
    from paper_2306_07629_b200 import DsqError
    with pytest.raises(DsqError) as e:
        _create(layer)
    return e.value.code


@pytest.fixture()
def good():
    return to_quantized_layer(make_layer(40, 70, 3, 0.02, seed=9))


def test_validation_empty_name(good):
    good.name = ""
    assert _errc(good) == 11  # invalid_argument (packfmt.cpp:83)


def test_validation_bits(good):
    good.packed.bits = 9
    assert _errc(good) == 11  # packfmt.cpp:8


def test_validation_payload_len(good):
    good.packed.payload = good.packed.payload[:-1]
    assert _errc(good) == 9  # shape_mismatch (packfmt.cpp:14-15)


def test_validation_groups(good):
    good.packed.groups_per_row = 3  # does not divide 70
    assert _errc(good) == 9


def test_validation_csr_cols_overflow():
    L = to_quantized_layer(make_layer(4, 8, 3, 0.0, seed=1))
    L.sparse.cols = 70000
    assert _errc(L) == 5  # dimension_overflow (dns.cpp:11)


def test_validation_csr_order(good):
    s = good.sparse
    r = int(np.argmax(np.diff(s.row_ptr.astype(np.int64))))
    a, b = int(s.row_ptr[r]), int(s.row_ptr[r + 1])
    assert b - a >= 2
    s.col_idx = s.col_idx.copy()
    s.col_idx[a], s.col_idx[a + 1] = s.col_idx[a + 1], s.col_idx[a]
    assert _errc(good) == 15  # internal: not strictly increasing (dns.cpp:20-23)


def test_validation_nonfinite(good):
    good.sparse.values = good.sparse.values.astype(np.float32)
    good.sparse.values[0] = np.nan
    assert _errc(good) == 3  # non_finite_value (dns.cpp:26-28)


def test_validation_dims(good):
    good.rows = 41
    assert _errc(good) == 9


def test_grouped_luts_pass_validation():
    """groups_per_row > 1 (the grouping ablation) is a valid device layer now
    (grouped_gemv); on a host without a GPU the upload then fails with
    no_device, never with unsupported / shape_mismatch."""
    from conftest import has_gpu
    from paper_2306_07629_b200 import DeviceLayer
    L = to_quantized_layer(make_layer(4, 64, 3, 0.0, seed=2, groups=2))
    assert L.packed.groups_per_row == 2
    if has_gpu():
        assert DeviceLayer(L).info().groups_per_row == 2
    else:
        assert _errc(L) == 101


def test_no_gpu_fails_loudly(good):
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("GPU present")
    assert _errc(good) == 101  # no_device: no silent CPU fallback


def test_x_dimension_mismatch_raises(good):
    from paper_2306_07629_b200 import DsqError, fused_dns_matvec
    with pytest.raises(DsqError) as e:
        fused_dns_matvec(good, np.zeros(good.cols + 1, np.float32))
    assert e.value.code == 9 and e.value.classify() == "argument"
