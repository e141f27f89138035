"""Whole-model decode stacks on one GPU (BASELINE configs[2] and the TP=1 leg
of configs[3]): LLaMA-7B/13B/65B-shaped linear stacks, 3-bit LUT + 0.45% CSR,
batch 1, run by the persistent stack kernel -- every GEMV of every decoder
layer of `--tokens` decode steps in ONE launch, chained like the bench
(v,q,k <- previous down; o <- v; up,gate <- o; down <- up).

Prints one JSON line per model: µs per GEMV, decode tok/s of the linear
stack, effective GB/s (reference-charged bytes) and its fraction of the copy
peak.  Weights rotate over `--rotation` distinct device copies of one decoder
layer (working set >> L2).  Synthetic layers are generated directly in the
packed layout (uniformly random 3-bit indices are uniformly random payload
bytes; CSR positions are cleared to index 0 as quantize_layer does,
pipeline.cpp:25-32) so 65B shapes build in seconds.

Under torchrun (WORLD_SIZE > 1, one process per GPU) the model runs
tensor-parallel (configs[3]): v,q,k,up,gate column-parallel, o,down
row-parallel, the two all-reduces per decoder layer fused into the stack
kernel over NVLink peer memory; timing is the max over ranks.

usage: python tools/bench_stack.py [--model 13b] [--tokens 3] [--rotation 8] [--batch 1..16]
       torchrun --nproc-per-node 8 tools/bench_stack.py --model 65b
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

MODELS = {  # hidden, intermediate, decoder layers
    "7b": (4096, 11008, 32),
    "13b": (5120, 13824, 40),
    "65b": (8192, 22016, 80),
}


def shapes(h, f):
    # the decoder launch order of paper_2306_07629_b200.tp.DECODER
    return [("v", h, h), ("q", h, h), ("o", h, h), ("k", h, h), ("up", f, h), ("gate", f, h),
            ("down", h, f)]


SPARSITY_ARG = 0.0045  # --sparsity


def fast_layer(rows, cols, bits=3, sparsity=0.0045, seed=0):
    from paper_2306_07629_b200 import CsrMatrix, PackedDense, QuantizedLayer
    from oracle.oracle import nnz_for
    rng = np.random.default_rng(seed)
    k = 1 << bits
    stride = (cols * bits + 7) // 8
    payload = rng.integers(0, 256, size=rows * stride, dtype=np.uint8)
    luts = np.sort(rng.normal(0.0, 0.02, size=(rows, k)).astype(np.float16), axis=1).reshape(-1)
    nnz = nnz_for(rows * cols, sparsity)
    pos = np.unique(rng.integers(0, rows * cols, size=nnz, dtype=np.int64))
    r, c = pos // cols, pos % cols
    # clear the packed index bits of the outlier positions (index 0)
    for b in range(bits):
        bitpos = r * stride * 8 + c * bits + b
        np.bitwise_and.at(payload, bitpos >> 3, np.uint8(0xff) ^ (np.uint8(1) << (bitpos & 7).astype(np.uint8)))
    row_ptr = np.zeros(rows + 1, np.uint32)
    np.add.at(row_ptr, r + 1, 1)
    row_ptr = np.cumsum(row_ptr, dtype=np.uint64).astype(np.uint32)
    vals = rng.normal(0.0, 0.2, size=pos.size).astype(np.float16)
    packed = PackedDense(bits, rows, cols, luts, payload)
    sparse = CsrMatrix(rows, cols, row_ptr, c.astype(np.uint16), vals)
    return QuantizedLayer(f"{rows}x{cols}", rows, cols, packed, sparse, 10), int(pos.size)


def run(model, tokens, rotation, peak, rank=0, world=1, batch=1):
    import torch
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from paper_2306_07629_b200.dsq import TPContext
    from paper_2306_07629_b200.tp import decoder_chain, shard_decoder
    from oracle.oracle import make_x
    h, f, nl = MODELS[model]
    shp = shapes(h, f)
    t0 = time.time()
    cache, qls, nnzs = {}, [], []
    for name, r, c in shp:
        if (r, c) not in cache:
            cache[(r, c)] = fast_layer(r, c, sparsity=SPARSITY_ARG, seed=r * 7 + c)
        q, nz = cache[(r, c)]
        qls.append(q)
        nnzs.append(nz)
    bytes_dec = sum(int(N.lib.dsq_bytes_touched_estimate(r, c, 3, 0, nz))
                    for (_, r, c), nz in zip(shp, nnzs))
    shards = shard_decoder(qls, rank, world) if world > 1 else qls
    dev = torch.cuda.current_device()
    dls = [[DeviceLayer(q, device=dev) for q in shards] for _ in range(rotation)]
    # batch B: B sequences decoded together, vector v at +v * stride
    YS = max(h, f)
    x = torch.from_numpy(np.tile(make_x(h), batch).view(np.int16)).cuda()
    ys = [[torch.empty(q.rows * batch if batch == 1 else YS * batch, dtype=torch.int16,
                       device="cuda") for q in shards]
          for _ in range(rotation)]
    tp = None
    if world > 1:
        import torch.distributed as dist
        tp = TPContext(world, rank, max_rows=h,
                       max_grid=torch.cuda.get_device_properties(dev).multi_processor_count,
                       device=dev)
        handles = [None] * world
        dist.all_gather_object(handles, tp.ipc_handle)
        tp.connect(handles)
    setup = time.time() - t0

    def build(ntok):
        deps, reduce, _ = decoder_chain(ntok * nl, 1)
        layers, yp = [], []
        for t in range(ntok * nl):
            slot = t % rotation
            layers += dls[slot]
            yp += [y.data_ptr() for y in ys[slot]]
        xp = [x.data_ptr() if d < 0 else 0 for d in deps]
        if batch > 1:
            return DeviceStack(layers, deps, xp, yp, N.F16, batch=batch, x_stride=h, y_stride=YS)
        if tp is None:
            return DeviceStack(layers, deps, xp, yp, N.F16)
        return DeviceStack(layers, deps, xp, yp, N.F16, reduce=reduce, tp=tp)

    warm, timed = build(1), build(tokens)
    warm.run(0)
    timed.run(0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    timed.run(0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tp.check()
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    gemvs = tokens * nl * 7
    gbs = bytes_dec * nl * tokens / (ms * 1e-3) / 1e9
    return {
        "model": f"llama-{model} linear stack ({nl} decoder layers x 7 GEMVs, 3-bit + 0.45% CSR)",
        "tokens": tokens, "gpus": world, "parallelism": f"tp{world}", "batch": batch,
        "form": "persistent" if timed.persistent else f"sequential ({timed.launches} launches)",
        "us_per_gemv": round(ms * 1e3 / gemvs, 3),
        "ms_per_token": round(ms / tokens, 4),
        "decode_tok_s_linear": round(batch * tokens / (ms * 1e-3), 1),
        "effective_GBs": round(gbs, 1), "frac_of_peak_per_gpu": round(gbs / world / peak, 4),
        "bytes_per_token": bytes_dec * nl, "rotation": rotation, "setup_s": round(setup, 1),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="13b", choices=list(MODELS) + ["all"])
    ap.add_argument("--tokens", type=int, default=3)
    ap.add_argument("--rotation", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1, help="sequences decoded together (1..16)")
    ap.add_argument("--sparsity", type=float, default=0.0045, help="CSR outlier density")
    args = ap.parse_args()
    global SPARSITY_ARG
    SPARSITY_ARG = args.sparsity
    try:
        peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        peak = 6650.0
    import os
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    for m in (list(MODELS) if args.model == "all" else [args.model]):
        line = run(m, args.tokens, args.rotation, peak, rank, world, args.batch)
        if rank == 0:
            print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
