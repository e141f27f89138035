"""`dsq profile` (reference tools/dsq.cpp:220-271) over the product's roofline
model, plus the hot-path table: per fused Dense-and-Sparse LUT-GEMV of a
LLaMA shape, the reference-charged bytes and the roofline-predicted time on
the B200 profile, beside a measured number when one is given.

usage: python tools/dsq_profile.py --hw data/b200.json --shape data/llama-7b.json \
           [--seq-len 2048] [--bits 3,4,8,16]
       python tools/dsq_profile.py --path [--model 7b] [--bits 3] [--sparsity 0.0045]
           [--measured profiles/r01_bench.json]
"""
import argparse
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

SHAPES = {"7b": (4096, 11008), "13b": (5120, 13824), "65b": (8192, 22016)}


def nnz_for(n, frac):  # dns.cpp:84-85 split of the 0.45% default (0.05% + 0.40%)
    return math.ceil(0.0005 * n) + math.ceil((frac - 0.0005) * n) if frac > 0 else 0


def path_table(model, bits, sparsity, hw, measured_us=None):
    from paper_2306_07629_b200 import roofline as R
    h, f = SHAPES[model]
    rows = [("q/k/v/o", h, h, 4), ("gate/up", f, h, 2), ("down", h, f, 1)]
    out = [f"# hardware\t{hw.name}\tmem_bandwidth\t{hw.mem_bandwidth:.6g}",
           "gemv\trows\tcols\tbits\tnnz\tbytes\tpredicted_us\tbound" +
           ("\tmeasured_us\tfrac_of_roofline" if measured_us else "")]
    tot_b = tot_t = 0.0
    for name, r, c, k in rows:
        nz = nnz_for(r * c, sparsity)
        cost = R.gemv_cost(r, c, bits, nz, hw)
        tot_b += k * cost.total_bytes()
        tot_t += k * cost.predicted_time
        out.append(f"{name}\t{r}\t{c}\t{bits}\t{nz}\t{int(cost.total_bytes())}\t"
                   f"{cost.predicted_time * 1e6:.3f}\t"
                   f"{'memory' if cost.memory_bound else 'compute'}")
    per_gemv = tot_t / 7 * 1e6
    line = (f"# decoder layer (7 GEMVs)\tbytes\t{int(tot_b)}\tpredicted_us\t{tot_t * 1e6:.3f}"
            f"\tper_gemv_us\t{per_gemv:.3f}")
    if measured_us:
        line += f"\tmeasured_per_gemv_us\t{measured_us:.3f}\tfrac\t{per_gemv / measured_us:.4f}"
    out.append(line)
    return "\n".join(out) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hw", default=None, help="hardware profile JSON (default: B200)")
    ap.add_argument("--shape", default=str(ROOT / "data" / "llama-7b.json"))
    ap.add_argument("--seq-len", type=int, default=0)
    ap.add_argument("--bits", default="3,4,8,16")
    ap.add_argument("--path", action="store_true", help="hot-path GEMV table")
    ap.add_argument("--model", default="7b", choices=list(SHAPES))
    ap.add_argument("--sparsity", type=float, default=0.0045)
    ap.add_argument("--measured", default=None, help="bench JSON line (ms_per_step, 7 GEMVs)")
    a = ap.parse_args()
    from paper_2306_07629_b200 import roofline as R
    hw = R.load_hardware_profile(a.hw) if a.hw else R.b200_profile()
    if a.path:
        meas = None
        if a.measured:
            j = json.loads(Path(a.measured).read_text().strip().splitlines()[-1])
            meas = float(j["ms_per_step"]) * 1e3 / 7
        sys.stdout.write(path_table(a.model, int(a.bits.split(",")[0]), a.sparsity, hw, meas))
        return
    shape = R.load_model_shape(a.shape)
    if a.seq_len > 0:
        shape.seq_len = a.seq_len
    sys.stdout.write(R.profile_report(hw, shape, [int(b) for b in a.bits.split(",")]))


if __name__ == "__main__":
    main()
