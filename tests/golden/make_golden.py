"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (needs oracle/_ref/libdsqref.so, which is compiled from the
unmodified sources under /root/reference/proj by oracle/Makefile):

    make -C oracle && python tests/golden/make_golden.py

Every expected output below is produced by the reference library
(dsq::lut_matvec / csr_matvec / fused_dns_matvec / ref::fused_dns_matvec /
ref::dequant_dense / pack / bytes_touched_estimate), never by our code.
Inputs are fp16-exact so the B200 path (fp16 storage) sees identical values.
The reference's own tests pin nothing on this path (proj/tests/test_kernels.cpp
and test_packfmt.cpp are one-line stubs; tests/golden/ is absent upstream,
SURVEY.md §4), so these files plus the SPEC.md KATs are the pins.
"""
from __future__ import annotations

import hashlib
import zlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Layer, Reference, make_layer, make_x  # noqa: E402

OUT = Path(__file__).resolve().parent

CASES = [
    # name, rows, cols, bits, sparsity, skew, seed
    ("l64x64_b3_s045_uniform", 64, 64, 3, 0.0045, "uniform", 11),
    ("l96x160_b4_s5_zipf", 96, 160, 4, 0.05, "zipf", 12),
    ("l48x256_b3_s2_halfrow", 48, 256, 3, 0.02, "halfrow", 13),
    ("l33x70_b5_s1_ragged", 33, 70, 5, 0.01, "uniform", 14),
    ("l40x96_b2_dense", 40, 96, 2, 0.0, "uniform", 15),
    ("l32x128_b8_s045", 32, 128, 8, 0.0045, "uniform", 16),
]


def student_t(rng, shape, nu=4):
    z = rng.normal(size=shape)
    chi2 = (rng.normal(size=(nu,) + shape) ** 2).sum(axis=0)
    return z / np.sqrt(chi2 / nu)


def quantized_case(ref: Reference, rows=64, cols=256, bits=3, sparsity=0.0045, seed=42):
    """The reference's own producer (quantize_layer, pipeline.cpp:7-47) on a
    Student-t matrix (the dsq_bench.cpp:23-62 recipe), then LUTs/deltas rounded
    to fp16 so the fixture is device-exact; outputs recomputed by the reference
    on the rounded layer."""
    rng = np.random.default_rng(seed)
    w = student_t(rng, (rows * cols,)).astype(np.float32)
    sens = rng.uniform(size=rows * cols).astype(np.float32)
    q = ref.quantize(w, sens, rows, cols, bits, sparsity / 9.0, sparsity - sparsity / 9.0,
                     top_k=10, seed=seed)
    a = q.arrays()
    luts16 = a["luts"].astype(np.float16)
    # LUT rounding may break the sorted/duplicate-free property; the kernels
    # do not rely on it (codebooks may repeat, nuq.hpp:16-17)
    vals16 = a["values"].astype(np.float16)
    payload = a["payload"]
    # recover the assignment from the payload with the reference unpack
    rc, assign = ref.unpack(payload, bits, rows, cols)
    assert rc == 0
    return Layer(bits, rows, cols, assign, luts16, payload, a["row_ptr"], a["col_idx"], vals16)


def dump(name: str, L: Layer, ref: Reference, manifest: dict):
    x = make_x(L.cols, seed=zlib.crc32(name.encode()) % 1000)
    x32 = x.astype(np.float32)
    rl = ref.layer(L, top_k=10)
    rc, repacked = ref.pack(L.assign, L.luts32, L.bits, L.rows, L.cols)
    assert rc == 0 and np.array_equal(repacked, L.payload)
    out = dict(
        bits=np.int64(L.bits), rows=np.int64(L.rows), cols=np.int64(L.cols),
        assign=L.assign, luts16=L.luts16, payload=L.payload, row_ptr=L.row_ptr,
        col_idx=L.col_idx, values16=L.values16, x16=x,
        y_lut=rl.matvec("lut", x32), y_csr=rl.matvec("csr", x32),
        y_fused=rl.matvec("fused", x32), y_fused_serial=rl.matvec("fused", x32, parallel=False),
        y_ref_fused=rl.matvec("reference", x32), dequant=rl.dequant_dense(),
        bytes_touched=np.int64(rl.bytes_touched()),
    )
    path = OUT / f"{name}.npz"
    np.savez_compressed(path, **out)
    manifest[name] = hashlib.sha256(path.read_bytes()).hexdigest()


def main():
    ref = Reference()
    manifest = {}
    # SPEC.md:347-348 pack KATs, produced by the reference pack()
    kat = {}
    rc, p3 = ref.pack(np.array([1, 2, 3], np.uint16), np.zeros(8, np.float32), 3, 1, 3)
    kat["pack3_123"] = p3.tobytes().hex()
    rc, p4 = ref.pack(np.arange(16, dtype=np.uint16), np.zeros(16, np.float32), 4, 1, 16)
    kat["pack4_0_15"] = p4.tobytes().hex()
    (OUT / "pack_kat.json").write_text(json.dumps(kat, indent=1) + "\n")
    for name, rows, cols, bits, sp, skew, seed in CASES:
        dump(name, make_layer(rows, cols, bits, sp, seed=seed, skew=skew), ref, manifest)
    dump("quantized_64x256_b3_s045", quantized_case(ref), ref, manifest)
    dump("quantized_32x128_b4_s045", quantized_case(ref, 32, 128, 4, 0.0045, 43), ref, manifest)
    (OUT / "MANIFEST.json").write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")
    print(json.dumps(kat), len(manifest), "fixtures")


if __name__ == "__main__":
    main()
