"""GPU channel-wise quantization (K9) vs the reference's CPU
quantize_channelwise on a LLaMA-7B-shaped layer (Student-t weights, squared-
normal sensitivities, 3-bit weighted k-means, 0.45% of positions masked as
extracted outliers).  The reference runs on a bounded row sample with all
host threads and is scaled to the full layer; the GPU quantizes the whole
layer (host arrays in/out, as the C ABI does).  Codebooks of the sampled rows
are compared bit for bit.

usage: python tools/quantize_bench.py [--rows 4096] [--cols 4096] [--ref-rows 64]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--bits", type=int, default=3)
    ap.add_argument("--ref-rows", type=int, default=64)
    a = ap.parse_args()
    from paper_2306_07629_b200.quantize import QuantConfig, quantize_channelwise
    from oracle.oracle import Reference
    rng = np.random.default_rng(0)
    w = (rng.standard_t(4, size=(a.rows, a.cols)) * 0.02).astype(np.float32)
    sens = (rng.normal(size=(a.rows, a.cols)) ** 2).astype(np.float32)
    mask = (rng.random(w.shape) < 0.0045).astype(np.uint8)  # stand-in for the extracted set
    cfg = QuantConfig(bits=a.bits)
    quantize_channelwise(w[:8], sens[:8], cfg, mask=mask[:8])  # warm-up (context, module load)
    t0 = time.perf_counter()
    res = quantize_channelwise(w, sens, cfg, mask=mask)
    gpu_s = time.perf_counter() - t0
    ref = Reference()
    threads = int(ref.lib.ref_max_threads())
    rr = min(a.ref_rows, a.rows)
    t0 = time.perf_counter()
    rc, cent, assign, _, _ = ref.quantize_channelwise(w[:rr], sens[:rr], a.bits, mask=mask[:rr])
    ref_s = (time.perf_counter() - t0) * a.rows / rr
    same = rc == 0 and np.array_equal(cent.view(np.uint32), res.codebooks[:rr].view(np.uint32)) \
        and np.array_equal(assign, res.assignment[:rr])
    # the whole pipeline (decompose + k-means + pack + CSR deltas) on the GPU
    from paper_2306_07629_b200.quantize import quantize_layer
    t0 = time.perf_counter()
    layer, stats = quantize_layer(w, sens, cfg)
    pipe_s = time.perf_counter() - t0
    print(json.dumps({
        "workload": f"quantize_channelwise {a.rows}x{a.cols} {a.bits}-bit weighted k-means",
        "gpu_s": round(gpu_s, 4), "reference_cpu_s_est": round(ref_s, 2),
        "reference_threads": threads, "reference_sample_rows": rr,
        "speedup": round(ref_s / gpu_s, 1), "sample_bit_identical": bool(same),
        "quantize_layer_gpu_s": round(pipe_s, 4), "quantize_layer_nnz": int(layer.sparse.row_ptr[-1]),
        "avg_bits": round(stats["avg_bits"], 4),
        "host_cores": os.cpu_count()}))


if __name__ == "__main__":
    main()
