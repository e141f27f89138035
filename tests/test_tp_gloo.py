"""Tensor-parallel sharding host logic (paper_2306_07629_b200.tp), world size 2
over torch.distributed gloo on CPU: column-parallel shards + all_gather and
row-parallel shards + all_reduce reproduce the unsharded reference product.
The per-shard product is the oracle (CPU); the GPU variant of the same
sharding is checked in test_gpu_parity-style below (single device)."""
import os
import socket

import numpy as np
import pytest

from oracle.oracle import Layer, make_layer, make_x, to_quantized_layer


def as_oracle_layer(q):
    p, s = q.packed, q.sparse
    return Layer(p.bits, q.rows, q.cols, np.zeros(1, np.uint16), np.asarray(p.luts, np.float16),
                 np.asarray(p.payload, np.uint8), np.asarray(s.row_ptr, np.uint32),
                 np.asarray(s.col_idx, np.uint16), np.asarray(s.values, np.float16))


def free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, mode, rows, cols, bits, out_path):
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle
    from paper_2306_07629_b200.tp import shard_cols, shard_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        L = make_layer(rows, cols, bits, 0.02, seed=77, skew="zipf")
        q = to_quantized_layer(L)
        x = make_x(cols, seed=5).astype(np.float32)
        if mode == "rows":
            sq, r0, r1 = shard_rows(q, rank, world)
            part = o.fused_dns_matvec(as_oracle_layer(sq), x, 10)
            # all_gather of the row slices (pad to equal length)
            n = torch.tensor([r1 - r0])
            sizes = [torch.zeros(1, dtype=torch.long) for _ in range(world)]
            dist.all_gather(sizes, n)
            m = max(int(t) for t in sizes)
            buf = torch.zeros(m, dtype=torch.float64)
            buf[: r1 - r0] = torch.from_numpy(part)
            got = [torch.zeros(m, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(got, buf)
            y = np.concatenate([g[: int(s)].numpy() for g, s in zip(got, sizes)])
        else:
            sq, c0, c1 = shard_cols(q, rank, world)
            part = o.fused_dns_matvec(as_oracle_layer(sq), x[c0:c1], 10)
            t = torch.from_numpy(part.copy())
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            y = t.numpy()
        if rank == 0:
            np.save(out_path, y)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,rows,cols,bits", [("rows", 97, 256, 3), ("cols", 64, 320, 3),
                                                 ("cols", 40, 200, 4), ("rows", 33, 64, 4)])
def test_tp_world2_matches_unsharded(tmp_path, oracle, mode, rows, cols, bits):
    import torch.multiprocessing as mp
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(2, free_port(), mode, rows, cols, bits, out), nprocs=2, join=True)
    y = np.load(out)
    L = make_layer(rows, cols, bits, 0.02, seed=77, skew="zipf")
    x = make_x(cols, seed=5).astype(np.float32)
    ref = oracle.fused_dns_matvec(L, x, 10)
    if mode == "rows":
        assert np.array_equal(y, ref)  # rows are independent: bit-exact
    else:
        np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_shard_cols_repack_roundtrip(oracle):
    """Column shards re-pack the reference layout exactly (unpack of the shard
    == the column slice of the unpacked layer)."""
    from paper_2306_07629_b200.tp import shard_cols
    L = make_layer(50, 300, 3, 0.01, seed=3)
    q = to_quantized_layer(L)
    rc, full = oracle.unpack(L.payload, 3, 50, 300)
    full = full.reshape(50, 300)
    for world in (2, 3, 4):
        for r in range(world):
            sq, c0, c1 = shard_cols(q, r, world)
            rc, a = oracle.unpack(sq.packed.payload, 3, 50, c1 - c0)
            assert rc == 0
            assert np.array_equal(a.reshape(50, c1 - c0), full[:, c0:c1])
            assert c0 % 32 == 0


@pytest.mark.gpu
def test_tp_shards_on_device(oracle):
    """Every shard runs through the device path; recombined == unsharded."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2306_07629_b200 import fused_dns_matvec
    from paper_2306_07629_b200.tp import shard_cols, shard_rows
    L = make_layer(512, 1024, 3, 0.0045, seed=8)
    q = to_quantized_layer(L)
    x = make_x(1024, seed=9).astype(np.float32)
    ref = oracle.fused_dns_matvec(L, x, 10)
    for world in (2, 4, 8):
        y = np.concatenate([fused_dns_matvec(shard_rows(q, r, world)[0], x) for r in range(world)])
        assert np.abs(y - ref).max() <= 1e-5 * np.abs(ref).max()
        yc = np.zeros_like(ref)
        for r in range(world):
            sq, c0, c1 = shard_cols(q, r, world)
            yc += fused_dns_matvec(sq, x[c0:c1])
        assert np.abs(yc - ref).max() <= 1e-5 * np.abs(ref).max()


def test_decoder_shards_chain_locally():
    """The row split of every column-parallel producer equals the column split
    of its row-parallel consumer (o <- v, down <- up), so the fused-reduce
    stack needs no exchange before a row-parallel layer."""
    from paper_2306_07629_b200.tp import DECODER, decoder_chain, shard_decoder
    shp = {"v": (256, 256), "q": (256, 256), "k": (256, 256), "o": (256, 256),
           "up": (704, 256), "gate": (704, 256), "down": (256, 704)}
    qls = [to_quantized_layer(make_layer(*shp[n], 3, 0.01, seed=i), name=n)
           for i, n in enumerate(DECODER)]
    for world in (2, 4, 8):
        rows_v, rows_up, cols_o, cols_down = 0, 0, 0, 0
        ix = {n: i for i, n in enumerate(DECODER)}
        v, o, up, down = ix["v"], ix["o"], ix["up"], ix["down"]
        for r in range(world):
            s = shard_decoder(qls, r, world)
            assert s[o].cols == s[v].rows and s[down].cols == s[up].rows
            rows_v += s[v].rows
            rows_up += s[up].rows
            cols_o += s[o].cols
            cols_down += s[down].cols
            assert s[o].rows == 256 and s[down].rows == 256  # row-parallel: full outputs
        assert rows_v == cols_o == 256 and rows_up == cols_down == 704
    deps, reduce, _ = decoder_chain(2, 1)
    assert deps[:7] == [-1, -1, 0, -1, 2, 2, 4] and deps[7:14] == [6, 6, 7, 6, 9, 9, 11]
    assert [reduce[i] for i in range(7)] == [n in ("o", "down") for n in DECODER]
    assert [i for i, r in enumerate(reduce) if r] == [2, 6, 9, 13]


@pytest.mark.parametrize("bits,rows,cols,world", [(3, 40, 200, 2), (4, 33, 320, 3), (2, 17, 96, 4),
                                                  (5, 8, 250, 2), (8, 9, 64, 2)])
def test_shard_cols_repack_matches_oracle(oracle, bits, rows, cols, world):
    """dsq_shard_cols (C++) re-packs each column slice exactly like the
    reference pack() of the sliced indices; CSR entries filtered and rebased."""
    from paper_2306_07629_b200.tp import shard_cols, shard_rows, split_range
    L = make_layer(rows, cols, bits, 0.05, seed=rows * bits + cols, skew="zipf")
    q = to_quantized_layer(L)
    rc, assign = oracle.unpack(L.payload, bits, rows, cols)
    assert rc == 0
    idx = assign.reshape(rows, cols)
    for rank in range(world):
        sq, c0, c1 = shard_cols(q, rank, world, 8)
        assert (c0, c1) == split_range(cols, world, rank, 8)
        want = oracle.pack(np.ascontiguousarray(idx[:, c0:c1]).reshape(-1), bits, rows, c1 - c0)
        assert np.array_equal(np.asarray(sq.packed.payload), want)
        keep = (L.col_idx >= c0) & (L.col_idx < c1)
        assert np.array_equal(np.asarray(sq.sparse.col_idx), (L.col_idx[keep] - c0).astype(np.uint16))
        assert np.array_equal(np.asarray(sq.sparse.values), L.values16[keep])
        sr, r0, r1 = shard_rows(q, rank, world)
        assert np.array_equal(np.asarray(sr.packed.luts), L.luts16[r0 * (1 << bits):r1 * (1 << bits)])


def test_shard_decoder_roles():
    """v,q,k,up,gate split by rows, o and down by 32-aligned columns."""
    from paper_2306_07629_b200.tp import shard_decoder, split_range
    shapes = [(64, 96), (64, 96), (96, 64), (64, 96), (160, 96), (160, 96), (96, 160)]
    qs = [to_quantized_layer(make_layer(r, c, 3, 0.01, seed=i), name=f"l{i}")
          for i, (r, c) in enumerate(shapes)]
    for rank in range(2):
        out = shard_decoder(qs, rank, 2)
        for i, ((r, c), s) in enumerate(zip(shapes, out)):
            if i in (2, 6):
                lo, hi = split_range(c, 2, rank, 32)
                assert (s.rows, s.cols) == (r, hi - lo) and s.name.endswith(f".c{rank}")
            else:
                lo, hi = split_range(r, 2, rank, 32)
                assert (s.rows, s.cols) == (hi - lo, c) and s.name.endswith(f".r{rank}")


def test_split_range_and_shard_errors():
    """dsq_split_range covers [0, n) with aligned, ordered, disjoint pieces;
    the shard API rejects bad ranks and row-parallel grouped LUTs."""
    import pytest as _pytest
    from paper_2306_07629_b200 import DsqError
    from paper_2306_07629_b200.tp import shard_cols, split_range
    for n, world, align in [(4096, 8, 32), (22016, 8, 32), (11008, 3, 32), (100, 7, 1), (33, 4, 8)]:
        pieces = [split_range(n, world, r, align) for r in range(world)]
        assert pieces[0][0] == 0 and pieces[-1][1] == n
        for (a, b), (c, d) in zip(pieces, pieces[1:]):
            assert b == c and a <= b
        assert all(lo % align == 0 for lo, _ in pieces)
    with _pytest.raises(DsqError):
        split_range(64, 2, 2, 32)  # rank >= world
    q = to_quantized_layer(make_layer(8, 64, 3, 0.0, seed=1, groups=2))
    with _pytest.raises(DsqError) as e:
        shard_cols(q, 0, 2)
    assert e.value.code == 102  # unsupported: grouped LUTs are channel-wise only here
