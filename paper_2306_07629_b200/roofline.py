"""Roofline performance model: the reference's ``dsq`` roofline module
(include/dsq/roofline.hpp:10-88, src/roofline.cpp:10-209) and ``dsq profile``
(tools/dsq.cpp:220-271) over the C ABI (csrc/roofline.cpp), plus a B200
HardwareProfile and the per-GEMV prediction of the Dense-and-Sparse path
that bench.py prints beside the measured number.

    hw = b200_profile()                                # MEASURED_PEAKS.json or fallback
    shape = load_model_shape("data/llama-7b.json")
    dc = decode_step_costs(shape, hw)                  # per-layer LayerCost + total
    print(profile_report(hw, shape, [3, 4, 8, 16]))    # the `dsq profile` table
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path

from . import _native as N

ROOT = Path(__file__).resolve().parents[1]
KIND = {0: "fc", 1: "attn", 2: "other"}


@dataclass
class HardwareProfile:
    name: str
    peak_flops: float       # operations per second
    mem_bandwidth: float    # bytes per second

    def flops_per_byte(self) -> float:
        return self.peak_flops / self.mem_bandwidth

    def _c(self) -> N.HwProfile:
        return N.HwProfile(self.name.encode()[:63], self.peak_flops, self.mem_bandwidth)


@dataclass
class ModelShape:
    name: str
    num_layers: int
    hidden_dim: int
    ffn_dim: int
    num_heads: int
    vocab_size: int
    seq_len: int = 128
    weight_bits: int = 16
    activation_bits: int = 16

    def _c(self) -> N.ModelShape:
        return N.ModelShape(self.name.encode()[:63], self.num_layers, self.hidden_dim,
                            self.ffn_dim, self.num_heads, self.vocab_size, self.seq_len,
                            self.weight_bits, self.activation_bits)


@dataclass
class LayerCost:
    name: str
    kind: str
    flops: float
    weight_elems: float
    activation_elems: float
    weight_bytes: float
    activation_bytes: float
    predicted_time: float
    memory_bound: bool
    intensity: float

    def total_bytes(self) -> float:
        return self.weight_bytes + self.activation_bytes

    @classmethod
    def _from(cls, c: N.LayerCost) -> "LayerCost":
        return cls(c.name.decode(), KIND.get(c.kind, "other"), c.flops, c.weight_elems,
                   c.activation_elems, c.weight_bytes, c.activation_bytes, c.predicted_s,
                   bool(c.memory_bound), c.intensity)


@dataclass
class DecodeCosts:
    layers: list = field(default_factory=list)
    total: LayerCost | None = None
    weight_traffic_share: float = 0.0


def decode_step_costs(shape: ModelShape, hw: HardwareProfile) -> DecodeCosts:
    arr = (N.LayerCost * N.DECODE_COSTS)()
    tot = N.LayerCost()
    share = C.c_double()
    s, h = shape._c(), hw._c()
    N.check(N.lib.dsq_decode_step_costs(C.byref(s), C.byref(h), arr, C.byref(tot),
                                        C.byref(share)))
    return DecodeCosts([LayerCost._from(c) for c in arr], LayerCost._from(tot), share.value)


def arithmetic_intensity(cost: LayerCost) -> float:
    c = N.LayerCost(cost.name.encode()[:31], 0, cost.flops, cost.weight_elems,
                    cost.activation_elems, cost.weight_bytes, cost.activation_bytes, 0.0, 0, 0.0)
    out = C.c_double()
    N.check(N.lib.dsq_arithmetic_intensity(C.byref(c), C.byref(out)))
    return out.value


@dataclass
class RuntimePoint:
    bits: int
    seconds: float
    normalized: float


def predicted_runtime_curve(shape: ModelShape, hw: HardwareProfile,
                            bit_list: list[int]) -> list[RuntimePoint]:
    n = len(bit_list)
    b = (C.c_uint32 * max(n, 1))(*bit_list)
    sec, nrm = (C.c_double * max(n, 1))(), (C.c_double * max(n, 1))()
    s, h = shape._c(), hw._c()
    N.check(N.lib.dsq_predicted_runtime_curve(C.byref(s), C.byref(h), b, n, sec, nrm))
    return [RuntimePoint(bit_list[i], sec[i], nrm[i]) for i in range(n)]


def affine_fit_r2(pts: list[RuntimePoint]) -> float:
    n = len(pts)
    b = (C.c_uint32 * max(n, 1))(*[p.bits for p in pts])
    y = (C.c_double * max(n, 1))(*[p.normalized for p in pts])
    r2 = C.c_double()
    N.check(N.lib.dsq_affine_fit_r2(b, y, n, C.byref(r2)))
    return r2.value


def load_hardware_profile(path) -> HardwareProfile:
    h = N.HwProfile()
    N.check(N.lib.dsq_load_hardware_profile(str(path).encode(), C.byref(h)))
    return HardwareProfile(h.name.decode(), h.peak_flops, h.mem_bandwidth)


def load_model_shape(path) -> ModelShape:
    s = N.ModelShape()
    N.check(N.lib.dsq_load_model_shape(str(path).encode(), C.byref(s)))
    return ModelShape(s.name.decode(), s.num_layers, s.hidden_dim, s.ffn_dim, s.num_heads,
                      s.vocab_size, s.seq_len, s.weight_bits, s.activation_bits)


def b200_profile(measured_peaks=ROOT / "MEASURED_PEAKS.json") -> HardwareProfile:
    """B200 from the pool's measured copy bandwidth / bf16 throughput
    (MEASURED_PEAKS.json) or the profiling recipe's fallback."""
    h = N.HwProfile()
    p = str(measured_peaks).encode() if measured_peaks and Path(measured_peaks).exists() else None
    N.check(N.lib.dsq_hw_profile_b200(p, C.byref(h)))
    return HardwareProfile(h.name.decode(), h.peak_flops, h.mem_bandwidth)


def gemv_cost(rows: int, cols: int, bits: int, nnz: int, hw: HardwareProfile,
              batch: int = 1) -> LayerCost:
    """One fused Dense-and-Sparse LUT-GEMV: reference-charged bytes
    (kernels.cpp:205-212) and its roofline-predicted time on `hw`."""
    c = N.LayerCost()
    h = hw._c()
    N.check(N.lib.dsq_gemv_cost(rows, cols, bits, nnz, batch, C.byref(h), C.byref(c)))
    return LayerCost._from(c)


def _fmt(v: float) -> str:  # tools/dsq.cpp:30-34 (%.12g)
    return f"{v:.12g}"


def profile_report(hw: HardwareProfile, shape: ModelShape, bits: list[int]) -> str:
    """The `dsq profile` output (tools/dsq.cpp:226-269), same columns."""
    out = [f"# hardware\t{hw.name}\tpeak_flops\t{_fmt(hw.peak_flops)}\tmem_bandwidth\t"
           f"{_fmt(hw.mem_bandwidth)}\tflops_per_byte\t{_fmt(hw.flops_per_byte())}",
           f"# model\t{shape.name}\tseq_len\t{shape.seq_len}\tweight_bits\t{shape.weight_bits}",
           "layer\tkind\tflops\tweight_elems\tact_elems\tbytes\ttime_s\tbound\tintensity"]
    dc = decode_step_costs(shape, hw)
    for c in dc.layers + [dc.total]:
        out.append("\t".join([c.name, c.kind, _fmt(c.flops),
                              _fmt(c.weight_elems), _fmt(c.activation_elems),
                              _fmt(c.total_bytes()), _fmt(c.predicted_time),
                              "memory" if c.memory_bound else "compute",
                              _fmt(arithmetic_intensity(c))]))
    out.append(f"# weight_traffic_share\t{_fmt(dc.weight_traffic_share)}")
    out.append("# runtime_curve")
    out.append("bits\tseconds\tnormalized")
    for p in predicted_runtime_curve(shape, hw, bits):
        out.append(f"{p.bits}\t{_fmt(p.seconds)}\t{_fmt(p.normalized)}")
    return "\n".join(out) + "\n"
