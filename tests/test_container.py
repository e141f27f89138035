"""The container loader (dsq_container_check / dsq_cuda_container_open) vs
the reference's own save_container / load_container (container.cpp:146-223),
compiled from its sources (oracle/_ref): same accepted files, same meta, same
error codes on corrupted files, and (GPU) device products of the loaded
layers equal to the reference's products of ITS loaded layers."""
import ctypes as C
import struct

import numpy as np
import pytest

from oracle.oracle import make_layer, make_x

ERR = {"missing_file": 1, "malformed_header": 2, "truncated_payload": 6,
       "checksum_mismatch": 7, "unsupported_version": 8}


def _crc(b: bytes) -> int:
    import zlib
    return zlib.crc32(b) & 0xFFFFFFFF


def _save(reference, layers, path, bits=3):
    hs = [reference.layer(L, top_k=10) for L in layers]
    arr = (C.c_void_p * len(hs))(*[h.h.value for h in hs])
    rc = reference.lib.ref_save_container(arr, len(hs), bits, str(path).encode())
    assert rc == 0, reference.err()
    return hs


def _ref_load_rc(reference, path):
    h = C.c_void_p()
    return reference.lib.ref_load_container_layer(str(path).encode(), 0, C.byref(h))


@pytest.fixture()
def cont(reference, tmp_path):
    layers = [make_layer(33, 70, 3, 0.02, seed=1), make_layer(64, 256, 3, 0.0045, seed=2),
              make_layer(40, 96, 4, 0.01, seed=3, skew="halfrow")]
    p = tmp_path / "m.dsq"
    _save(reference, layers, p)
    return p, layers


def test_check_accepts_reference_file(cont):
    from paper_2306_07629_b200 import check_container
    p, layers = cont
    m = check_container(p)
    assert m["n_layers"] == len(layers) and m["bits"] == 3


def _mutate(src, dst, fn, fix_crc=True):
    raw = bytearray(src.read_bytes())
    raw = fn(raw)
    if fix_crc and len(raw) >= 16:
        raw[-4:] = struct.pack("<I", _crc(bytes(raw[12:-4])))
    dst.write_bytes(bytes(raw))


@pytest.mark.parametrize("case", ["missing", "small", "magic", "version", "crc", "truncated",
                                  "trailing", "bits", "payload_len"])
def test_error_codes_match_reference(reference, cont, tmp_path, case):
    from paper_2306_07629_b200 import DsqError, check_container
    p, _ = cont
    q = tmp_path / f"bad_{case}.dsq"
    if case == "missing":
        q = tmp_path / "nope.dsq"
    elif case == "small":
        q.write_bytes(b"DSQCONT1\x01\x00")
    elif case == "magic":
        _mutate(p, q, lambda r: bytearray(b"DSQCONT2") + r[8:])
    elif case == "version":
        _mutate(p, q, lambda r: r[:8] + bytearray(struct.pack("<I", 2)) + r[12:])
    elif case == "crc":
        _mutate(p, q, lambda r: r[:40] + bytearray([r[40] ^ 0xFF]) + r[41:], fix_crc=False)
    elif case == "truncated":
        _mutate(p, q, lambda r: r[:-200] + r[-4:])
    elif case == "trailing":
        _mutate(p, q, lambda r: r[:-4] + bytearray(b"\x00" * 8) + r[-4:])
    elif case == "bits":  # first layer bits field (after meta 52 B, n_layers, name)
        def f(r):
            nlen = struct.unpack_from("<I", r, 12 + 56)[0]
            off = 12 + 56 + 4 + nlen + 8
            r[off:off + 4] = struct.pack("<I", 9)
            return r
        _mutate(p, q, f)
    elif case == "payload_len":
        def f(r):
            nlen = struct.unpack_from("<I", r, 12 + 56)[0]
            off = 12 + 56 + 4 + nlen
            rows, cols, bits, groups = struct.unpack_from("<IIII", r, off)
            off += 16 + rows * groups * (1 << bits) * 4
            r[off:off + 8] = struct.pack("<Q", struct.unpack_from("<Q", r, off)[0] + 1)
            return r
        _mutate(p, q, f)
    with pytest.raises(DsqError) as e:
        check_container(q)
    ref_rc = _ref_load_rc(reference, q)
    assert ref_rc != 0
    assert e.value.code == ref_rc, (case, e.value.code, ref_rc, str(e.value))


@pytest.mark.gpu
def test_loaded_layers_match_reference_products(reference, cont):
    from paper_2306_07629_b200 import load_container
    import paper_2306_07629_b200._native as N
    p, layers = cont
    c = load_container(p)
    assert c.meta["n_layers"] == len(layers)
    for i, L in enumerate(layers):
        h = C.c_void_p()
        assert reference.lib.ref_load_container_layer(str(p).encode(), i, C.byref(h)) == 0
        from oracle.oracle import RefLayer
        rl = RefLayer(reference, h, L.rows, L.cols)
        x = make_x(L.cols, seed=i).astype(np.float32)
        want = rl.matvec("fused", x)
        got = c.layers[i].matvec_host(N.KERNEL_FUSED, x)
        info = c.layers[i].info()
        assert info.luts_exact_f16 and info.values_exact_f16
        scale = np.abs(want).max() + 1e-30
        assert np.abs(got - want).max() / scale <= 1e-3
