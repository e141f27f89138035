"""Pin the oracle (CPU, no GPU): SPEC.md known-answer vectors, the committed
golden fixtures produced by the reference, and bit-exact agreement of the C
restatement with the reference compiled from its own sources (oracle/_ref)."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Layer, make_layer, make_x

GOLDEN = Path(__file__).resolve().parent / "golden"
FIXTURES = sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load(name):
    z = np.load(GOLDEN / f"{name}.npz")
    L = Layer(int(z["bits"]), int(z["rows"]), int(z["cols"]), z["assign"], z["luts16"],
              z["payload"], z["row_ptr"], z["col_idx"], z["values16"])
    return L, z


# ---- SPEC.md known-answer tests -------------------------------------------
def test_pack_kat_3bit(oracle):
    # SPEC.md:347  bits=3, [1,2,3] -> [0xD1, 0x00]
    p = oracle.pack(np.array([1, 2, 3], np.uint16), 3, 1, 3)
    assert p.tobytes() == bytes([0xD1, 0x00])
    assert json.loads((GOLDEN / "pack_kat.json").read_text())["pack3_123"] == "d100"


def test_pack_kat_4bit(oracle):
    # SPEC.md:348  bits=4, 0..15 over 16 cols -> nibble i = i
    p = oracle.pack(np.arange(16, dtype=np.uint16), 4, 1, 16)
    assert p.tobytes().hex() == "1032547698badcfe"
    assert json.loads((GOLDEN / "pack_kat.json").read_text())["pack4_0_15"] == p.tobytes().hex()


def test_masked_index_packs_as_zero(oracle):
    # packfmt.cpp:47 kMaskedIndex (0xFFFF) -> 0
    p = oracle.pack(np.array([0xFFFF, 1, 0xFFFF], np.uint16), 3, 1, 3)
    rc, a = oracle.unpack(p, 3, 1, 3)
    assert rc == 0 and a.tolist() == [0, 1, 0]


def test_unpack_strict_rejects_pad_bits(oracle):
    # packfmt.cpp:71-77
    rc, _ = oracle.unpack(np.array([0xD1, 0x80], np.uint8), 3, 1, 3, strict=True)
    assert rc == 6  # truncated_payload
    rc, a = oracle.unpack(np.array([0xD1, 0x80], np.uint8), 3, 1, 3, strict=False)
    assert rc == 0 and a.tolist() == [1, 2, 3]


def _tiny(bits, rows, cols, assign, luts, row_ptr=None, col_idx=(), vals=()):
    from oracle.oracle import Oracle
    o = Oracle()
    payload = o.pack(np.asarray(assign, np.uint16), bits, rows, cols)
    rp = np.zeros(rows + 1, np.uint32) if row_ptr is None else np.asarray(row_ptr, np.uint32)
    return Layer(bits, rows, cols, np.asarray(assign, np.uint16), np.asarray(luts, np.float16),
                 payload, rp, np.asarray(col_idx, np.uint16), np.asarray(vals, np.float16))


def test_lut_matvec_kat(oracle):
    # 1x3, bits 2, lut [0,1,2,3], idx [1,2,3], x=1 -> 6 ; x=0 -> 0
    L = _tiny(2, 1, 3, [1, 2, 3], [0, 1, 2, 3])
    assert oracle.lut_matvec(L, np.ones(3, np.float32)).tolist() == [6.0]
    assert oracle.lut_matvec(L, np.zeros(3, np.float32)).tolist() == [0.0]


def test_csr_kats(oracle):
    # empty CSR -> 0 ; identity pattern -> x
    n = 5
    x = np.arange(1, n + 1, dtype=np.float32)
    L0 = _tiny(2, n, n, [0] * n * n, [0] * 4 * n)
    assert oracle.csr_matvec(L0, x).tolist() == [0.0] * n
    Li = _tiny(2, n, n, [0] * n * n, [0] * 4 * n, row_ptr=range(n + 1), col_idx=range(n),
               vals=[1.0] * n)
    assert oracle.csr_matvec(Li, x).tolist() == x.tolist()


def test_empty_sparse_fused_equals_lut(oracle):
    # SPEC.md:421
    L = make_layer(64, 96, 3, 0.0, seed=3)
    x = make_x(96).astype(np.float32)
    assert np.array_equal(oracle.fused_dns_matvec(L, x, 0), oracle.lut_matvec(L, x))


def test_hybrid_equivalence(oracle):
    # fused identical whether 0 or top_k rows are promoted
    L = make_layer(128, 256, 3, 0.02, seed=5, skew="zipf")
    x = make_x(256).astype(np.float32)
    assert np.array_equal(oracle.fused_dns_matvec(L, x, 0), oracle.fused_dns_matvec(L, x, 10))


def test_pack_unpack_property(oracle, reference):
    # unpack(pack(a)) == a for bits 2..8 (1000 cases), and the
    # restatement packs byte-identically to the reference pack()
    rng = np.random.default_rng(0)
    for i in range(1000):
        bits = int(rng.integers(2, 9))
        rows, cols = int(rng.integers(1, 5)), int(rng.integers(1, 40))
        a = rng.integers(0, 1 << bits, size=rows * cols, dtype=np.uint16)
        p = oracle.pack(a, bits, rows, cols)
        rc, b = oracle.unpack(p, bits, rows, cols)
        assert rc == 0 and np.array_equal(a, b)
        if i % 10 == 0:
            rc, pr = reference.pack(a, np.zeros(rows << bits, np.float32), bits, rows, cols)
            assert rc == 0 and np.array_equal(p, pr)


def test_csr_validate_codes(oracle):
    # dns.cpp:10-29 error codes
    rp = np.array([0, 2], np.uint32)
    ok = oracle.csr_validate(1, 10, rp, np.array([1, 3], np.uint16), np.ones(2, np.float32))
    assert ok == 0
    assert oracle.csr_validate(1, 70000, rp, np.array([1, 3], np.uint16),
                               np.ones(2, np.float32)) == 5
    assert oracle.csr_validate(1, 10, rp, np.array([3, 1], np.uint16),
                               np.ones(2, np.float32)) == 15
    assert oracle.csr_validate(1, 10, rp, np.array([1, 3], np.uint16),
                               np.array([1, np.inf], np.float32)) == 3


# ---- accounting -------------------------------------------------------------
@pytest.mark.parametrize("rows,cols,bits,nnz,expect", [
    (4096, 4096, 4, 0, 8_536_064),
    (4096, 4096, 3, 75_498, 6_691_756),   # config 2
    (11008, 4096, 3, 202_901, 17_970_264),
    (4096, 11008, 3, 202_901, 17_832_024),
])
def test_bytes_touched(oracle, rows, cols, bits, nnz, expect):
    assert oracle.bytes_touched(rows, cols, bits, 0, nnz) == expect


def test_avg_bits_spec_example(oracle):
    # SPEC.md packfmt: bits=3, square 4096, channel-wise -> 3 + 128/4096
    tb = oracle.layer_total_bits(4096, 4096, 3, 0, 0)
    assert tb / (4096 * 4096) == pytest.approx(3 + 128 / 4096)


def test_nnz_split_matches_reference_decompose():
    # dns.cpp:84-85 (ceil(sens*N) + ceil(out*N)) at the BASELINE shapes
    from oracle.oracle import nnz_for
    assert nnz_for(4096 * 4096, 0.0045) == 75_498
    assert nnz_for(4096 * 11008, 0.0045) == 202_901
    assert nnz_for(8192 * 22016, 0.0045) == 811_599


# ---- golden fixtures (produced by the reference) ---------------------------
def test_golden_manifest():
    man = json.loads((GOLDEN / "MANIFEST.json").read_text())
    assert sorted(man) == FIXTURES
    for name, sha in man.items():
        assert hashlib.sha256((GOLDEN / f"{name}.npz").read_bytes()).hexdigest() == sha


@pytest.mark.parametrize("name", FIXTURES)
def test_restatement_matches_golden(oracle, name):
    L, z = load(name)
    x = z["x16"].astype(np.float32)
    assert np.array_equal(oracle.pack(L.assign, L.bits, L.rows, L.cols), L.payload)
    assert np.array_equal(oracle.lut_matvec(L, x), z["y_lut"])
    assert np.array_equal(oracle.csr_matvec(L, x), z["y_csr"])
    assert np.array_equal(oracle.fused_dns_matvec(L, x, 10), z["y_fused"])
    assert np.array_equal(oracle.fused_dns_matvec(L, x, 10), z["y_fused_serial"])
    assert np.array_equal(oracle.dequant_dense(L), z["dequant"])
    assert oracle.bytes_touched(L.rows, L.cols, L.bits, 0, L.nnz) == int(z["bytes_touched"])
    # ref::fused_dns_matvec (dequantize-then-multiply) agrees to rounding
    np.testing.assert_allclose(z["y_ref_fused"], z["y_fused"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("rows,cols,bits,sp,skew", [
    (128, 256, 3, 0.0045, "uniform"), (64, 512, 4, 0.02, "zipf"),
    (200, 96, 3, 0.05, "halfrow"), (17, 45, 6, 0.01, "uniform"), (32, 64, 1, 0.0, "uniform"),
])
def test_restatement_matches_reference_live(oracle, reference, rows, cols, bits, sp, skew):
    L = make_layer(rows, cols, bits, sp, seed=rows + cols, skew=skew)
    x = make_x(cols, seed=cols).astype(np.float32)
    rl = reference.layer(L)
    assert np.array_equal(rl.matvec("lut", x), oracle.lut_matvec(L, x, nthreads=4))
    assert np.array_equal(rl.matvec("csr", x), oracle.csr_matvec(L, x))
    assert np.array_equal(rl.matvec("fused", x), oracle.fused_dns_matvec(L, x, 10, nthreads=4))
    assert np.array_equal(rl.dequant_dense(), oracle.dequant_dense(L))


@pytest.mark.parametrize("rows,cols,bits,groups", [(16, 128, 3, 4), (9, 96, 4, 2), (5, 64, 2, 8),
                                                   (7, 120, 5, 3)])
def test_grouped_restatement_matches_reference(oracle, reference, rows, cols, bits, groups):
    """Grouped LUTs (lut_at(r, c) = luts[(r*groups + c/gcols)*K], packfmt.hpp:28-31):
    the restated products and dequant equal the compiled reference bit for bit."""
    import ctypes as C
    L = make_layer(rows, cols, bits, 0.02, seed=rows * groups + bits, groups=groups)
    x = make_x(cols, seed=3).astype(np.float32)
    rl = reference.layer(L)
    assert np.array_equal(rl.matvec("lut", x), oracle.lut_matvec(L, x))
    assert np.array_equal(rl.matvec("fused", x), oracle.fused_dns_matvec(L, x, 10))
    assert np.array_equal(rl.dequant_dense(), oracle.dequant_dense(L))
    want = np.zeros(rows * cols, np.float32)
    assert reference.lib.ref_dequantize_layer(rl.h, C.c_void_p(want.ctypes.data)) == 0
