"""Roofline model: the product's C-ABI implementation
(csrc/roofline.cpp) against the UNMODIFIED reference module compiled here
(oracle/_ref/libdsqref_roofline.so: src/roofline.cpp + oracle/ref_roofline_shim.cpp),
value for value (the doubles are compared for equality), plus the SPEC.md
roofline examples and the hot-path GEMV byte charge."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2306_07629_b200 import _native as N
from paper_2306_07629_b200 import roofline as R

ROOT = Path(__file__).resolve().parents[1]
REFLIB = ROOT / "oracle" / "_ref" / "libdsqref_roofline.so"
DATA = ROOT / "data"
FIELDS = ["flops", "weight_elems", "activation_elems", "weight_bytes", "activation_bytes",
          "predicted_time"]
KINDS = {0: "fc", 1: "attn", 2: "other"}


@pytest.fixture(scope="module")
def ref():
    if not REFLIB.exists():
        pytest.skip("reference roofline not built (oracle/_ref absent)")
    lib = C.CDLL(str(REFLIB))
    u32p, dp = C.POINTER(C.c_uint32), C.POINTER(C.c_double)
    lib.dsqref_decode_step_costs.argtypes = [u32p, C.c_double, C.c_double, dp, C.c_uint32, u32p, dp]
    lib.dsqref_runtime_curve.argtypes = [u32p, C.c_double, C.c_double, u32p, C.c_uint32, dp, dp]
    lib.dsqref_affine_fit_r2.argtypes = [u32p, dp, C.c_uint32, dp]
    lib.dsqref_arithmetic_intensity.argtypes = [C.c_double, C.c_double, C.c_double, dp]
    lib.dsqref_load_hardware_profile.argtypes = [C.c_char_p, dp, dp]
    lib.dsqref_load_model_shape.argtypes = [C.c_char_p, u32p]
    return lib


def _shape_arr(s):
    return (C.c_uint32 * 7)(s.num_layers, s.hidden_dim, s.ffn_dim, s.num_heads, s.vocab_size,
                            s.seq_len, s.weight_bits)


SHAPES = ["llama-7b", "llama-13b", "llama-65b"]
HWS = ["a5000", "b200"]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("hw", HWS)
@pytest.mark.parametrize("seq_len,bits", [(128, 16), (2048, 16), (128, 3), (512, 4), (1, 8)])
def test_decode_step_costs_equal_reference(ref, shape, hw, seq_len, bits):
    s = R.load_model_shape(DATA / f"{shape}.json")
    s.seq_len, s.weight_bits = seq_len, bits
    h = R.load_hardware_profile(DATA / f"{hw}.json")
    dc = R.decode_step_costs(s, h)
    out = (C.c_double * (8 * 16))()
    n, share = C.c_uint32(), C.c_double()
    assert ref.dsqref_decode_step_costs(_shape_arr(s), h.peak_flops, h.mem_bandwidth, out, 16,
                                        C.byref(n), C.byref(share)) == 0
    assert n.value == len(dc.layers) == N.DECODE_COSTS
    got = np.frombuffer(out, dtype=np.float64).reshape(16, 8)
    for i, c in enumerate(dc.layers + [dc.total]):
        want = got[i]
        assert [getattr(c, f) for f in FIELDS] == list(want[:6]), (c.name, i)
        assert c.memory_bound == bool(want[6]) and c.kind == KINDS[int(want[7])]
    assert dc.weight_traffic_share == share.value


@pytest.mark.parametrize("shape", SHAPES)
def test_runtime_curve_and_fit_equal_reference(ref, shape):
    s = R.load_model_shape(DATA / f"{shape}.json")
    h = R.load_hardware_profile(DATA / "a5000.json")
    bits = list(range(2, 17))
    pts = R.predicted_runtime_curve(s, h, bits)
    b = (C.c_uint32 * len(bits))(*bits)
    sec, nrm = (C.c_double * len(bits))(), (C.c_double * len(bits))()
    assert ref.dsqref_runtime_curve(_shape_arr(s), h.peak_flops, h.mem_bandwidth, b, len(bits),
                                    sec, nrm) == 0
    assert [p.seconds for p in pts] == list(sec) and [p.normalized for p in pts] == list(nrm)
    r2 = C.c_double()
    assert ref.dsqref_affine_fit_r2(b, nrm, len(bits), C.byref(r2)) == 0
    assert R.affine_fit_r2(pts) == r2.value


def test_intensity_equal_reference(ref):
    s = R.load_model_shape(DATA / "llama-7b.json")
    dc = R.decode_step_costs(s, R.b200_profile(None))
    for c in dc.layers + [dc.total]:
        v = C.c_double()
        assert ref.dsqref_arithmetic_intensity(c.flops, c.weight_elems, c.activation_elems,
                                               C.byref(v)) == 0
        assert R.arithmetic_intensity(c) == v.value == c.intensity


def _ref_code(rc):
    return 15 if rc == 100 else rc  # non-dsq exception -> internal (CLI exit 4)


def _err(fn, *a):
    try:
        fn(*a)
    except N.DsqError as e:
        return e.code
    return 0


def test_errors_match_reference(ref, tmp_path):
    # zero-flop layer / zero memory ops: invalid_argument
    z = R.LayerCost("z", "other", 0.0, 1.0, 1.0, 0, 0, 0, True, 0)
    v = C.c_double()
    assert _err(R.arithmetic_intensity, z) == ref.dsqref_arithmetic_intensity(0.0, 1.0, 1.0,
                                                                              C.byref(v)) == 11
    # loaders: missing file, malformed JSON, missing key, bad shape values
    cases = {
        "missing": None,
        "malformed.json": "not json",
        "nokey.json": json.dumps({"name": "x", "peak_flops": 1e12}),
        "nameless.json": json.dumps({"peak_flops": 1e12, "mem_bandwidth_bytes_per_s": 1e9}),
        "neg.json": json.dumps({"name": "x", "peak_flops": -1, "mem_bandwidth_bytes_per_s": 1e9}),
    }
    for fname, text in cases.items():
        p = tmp_path / fname
        if text is not None:
            p.write_text(text)
        a, b = C.c_double(), C.c_double()
        want = _ref_code(ref.dsqref_load_hardware_profile(str(p).encode(), C.byref(a), C.byref(b)))
        assert _err(R.load_hardware_profile, p) == want, fname
    shapes = {
        "heads.json": {"name": "s", "num_layers": 2, "hidden_dim": 10, "ffn_dim": 4,
                       "num_heads": 3, "vocab_size": 5},
        "bits.json": {"name": "s", "num_layers": 2, "hidden_dim": 12, "ffn_dim": 4,
                      "num_heads": 3, "vocab_size": 5, "weight_bits": 1},
        "zero.json": {"name": "s", "num_layers": 0, "hidden_dim": 12, "ffn_dim": 4,
                      "num_heads": 3, "vocab_size": 5},
        "ok.json": {"name": "s", "num_layers": 2, "hidden_dim": 12, "ffn_dim": 4,
                    "num_heads": 3, "vocab_size": 5, "seq_len": 9},
    }
    for fname, d in shapes.items():
        p = tmp_path / fname
        p.write_text(json.dumps(d))
        arr = (C.c_uint32 * 7)()
        want = _ref_code(ref.dsqref_load_model_shape(str(p).encode(), arr))
        assert _err(R.load_model_shape, p) == want, fname
        if want == 0:
            s = R.load_model_shape(p)
            assert list(arr) == [s.num_layers, s.hidden_dim, s.ffn_dim, s.num_heads,
                                 s.vocab_size, s.seq_len, s.weight_bits]
    # curve with bits out of range
    s = R.load_model_shape(DATA / "llama-7b.json")
    assert _err(R.predicted_runtime_curve, s, R.b200_profile(None), [1]) == 11


def test_spec_examples():
    """SPEC.md:480-505 examples, on the paper's A5000 profile."""
    a5000 = R.load_hardware_profile(DATA / "a5000.json")
    assert round(a5000.flops_per_byte()) == 289  # "290x higher than its DRAM bandwidth"
    s = R.load_model_shape(DATA / "llama-7b.json")
    assert R.decode_step_costs(s, a5000).weight_traffic_share >= 0.99
    s.seq_len = 2048
    assert 0.94 <= R.decode_step_costs(s, a5000).weight_traffic_share <= 0.97
    s.seq_len = 128
    pts = R.predicted_runtime_curve(s, a5000, [4, 16])
    assert 0.24 <= pts[0].normalized <= 0.30
    assert R.affine_fit_r2(R.predicted_runtime_curve(s, a5000, list(range(3, 17)))) >= 0.999
    # matvec intensity is 2 per weight element (plus the activation elements)
    fc = R.decode_step_costs(s, a5000).layers[1]
    assert abs(R.arithmetic_intensity(fc) - 2.0) < 1e-3
    # doubling hidden_dim quadruples the square projections' flops and bytes
    s2 = R.ModelShape(**{**s.__dict__, "hidden_dim": 2 * s.hidden_dim})
    a, b = R.decode_step_costs(s, a5000).layers[1], R.decode_step_costs(s2, a5000).layers[1]
    assert b.flops == 4 * a.flops and b.weight_bytes == 4 * a.weight_bytes
    # pathological: tiny peak -> compute-bound, flat in bits
    slow = R.HardwareProfile("slow", 1.0, 1e12)
    pts = R.predicted_runtime_curve(s, slow, [3, 8, 16])
    assert all(p.normalized == 1.0 for p in pts)
    assert not R.decode_step_costs(s, slow).total.memory_bound


def test_gemv_cost_charges_reference_bytes():
    """The hot-path GEMV costs reference-charged bytes (kernels.cpp:205-212):
    the §8(d) figures for the LLaMA-7B shapes at 3-bit + 0.45%."""
    hw = R.b200_profile(None)
    assert hw.mem_bandwidth == 6.65e12 and "fallback" in hw.name
    for (r, c, nnz, want) in [(4096, 4096, 75498, 6691756), (11008, 4096, 202901, 17970264),
                              (4096, 11008, 202901, 17832024)]:
        g = R.gemv_cost(r, c, 3, nnz, hw)
        assert g.total_bytes() == want == N.lib.dsq_bytes_touched_estimate(r, c, 3, 0, nnz)
        assert g.memory_bound and g.predicted_time == want / hw.mem_bandwidth
    # batch B: weights once + B x/y vectors (§8d config 5)
    g1, g8 = R.gemv_cost(4096, 4096, 4, 0, hw), R.gemv_cost(4096, 4096, 4, 0, hw, batch=8)
    assert g8.total_bytes() - g1.total_bytes() == 7 * (4096 + 4096) * 2
    assert g8.flops == 8 * g1.flops


def test_b200_profile_reads_measured_peaks(tmp_path):
    p = tmp_path / "peaks.json"
    p.write_text(json.dumps({"hbm_gbs": 7000.0, "bf16_tflops": 1800.0}))
    hw = R.b200_profile(p)
    assert hw.mem_bandwidth == 7000e9 and hw.peak_flops == 1800e12 and "measured" in hw.name
