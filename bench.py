#!/usr/bin/env python
"""bench.py -- SqueezeLLM Dense-and-Sparse LUT-GEMV hot path on B200.

Workload (BASELINE.json configs[1], LLaMA-7B shapes, batch 1): one STEP is the
linear GEMV chain of one LLaMA-7B decoder layer, every GEMV a 3-bit LUT +
0.45% CSR fused product (the hot path):
    q,k,v,o : 4096 x 4096     gate,up : 11008 x 4096     down : 4096 x 11008
chained through fp16 outputs (v,q,k read the step input; o reads v; up,gate
read o; down reads up).  Each step uses a different decoder layer's weights out of a rotation
whose working set (>1 GB) is far larger than L2.

Steps are chained like consecutive decoder layers: the q/k/v input of step t
is the down output of step t-1 (attention, norms and residuals are out of
scope and are not computed).

  value  = effective HBM GB/s = reference-charged bytes of the 7 GEMVs
           (bytes_touched_estimate, kernels.cpp:205-212) / device time
  e2e    = same metric through the reference-facing host call
           (dsq_cuda_matvec_host: fp32 host x -> fp64 host y, per GEMV)
  --impl reference : the reference's own CPU fused_dns_matvec (compiled from
           /root/reference sources into oracle/_ref), all host threads.

Multi-GPU (torchrun, one process per GPU): replicas -- each rank streams its
own decoder layers (weak scaling, no data-path collective in this round).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LUT-GEMV µs/layer & effective HBM GB/s (% of peak); decode tok/s at 1/2/4/8"
# One decoder layer's GEMVs in dependency-aware issue order: v first so that o
# (which consumes the attention output, stood in for by v's output) does not
# wait; up before gate so that down (stand-in input: up's output) does not wait.
# launch order of one decoder layer's GEMVs: o (<- v) is placed between q
# and k so that k, which reads the step input, hides the o -> up/gate edge
# and q hides the v -> o edge (the persistent kernel runs layers in order)
SHAPES = [("v", 4096, 4096), ("q", 4096, 4096), ("o", 4096, 4096), ("k", 4096, 4096),
          ("up", 11008, 4096), ("gate", 11008, 4096), ("down", 4096, 11008)]
# input of each GEMV (index into this step's outputs; -1 = the step input,
# which is the previous step's down output -- steps chain like decoder layers)
CHAIN_IN = [-1, -1, 0, -1, 2, 2, 4]
BITS, SPARSITY = 3, 0.0045
LLAMA7B_LAYERS = 32


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def workload_config(n_rot: int, parallelism: str) -> dict:
    return {
        "workload": "llama7b-decoder-linear-chain: q,k,v,o 4096x4096; gate,up 11008x4096; "
                    "down 4096x11008; 3-bit LUT (8 fp16 centroids/row) + 0.45% CSR fp16 "
                    "outliers; batch 1 (BASELINE configs[1])",
        "gemvs_per_step": len(SHAPES),
        "bits": BITS, "sparsity": SPARSITY, "batch": 1,
        "l2": f"inputs larger than L2: rotation over {n_rot} decoder layers of distinct "
              f"device weights",
        "parallelism": parallelism,
    }


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[2:6]):
                    if v.strip().lower() in ("active", "1"):
                        reasons.add(n)
                pw.append(float(r[6]))
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------
# CPU (reference) leg
# ---------------------------------------------------------------------------
def slice_rows(L, r0, r1):
    from oracle.oracle import Layer
    k = 1 << L.bits
    stride = (L.cols * L.bits + 7) // 8
    a, b = int(L.row_ptr[r0]), int(L.row_ptr[r1])
    return Layer(L.bits, r1 - r0, L.cols, L.assign[r0 * L.cols:r1 * L.cols],
                 L.luts16[r0 * k:r1 * k], L.payload[r0 * stride:r1 * stride],
                 (L.row_ptr[r0:r1 + 1] - a).astype(np.uint32), L.col_idx[a:b],
                 L.values16[a:b])


def cpu_reference_sample(host_layers, frac: float, repeats: int = 3):
    """Time the reference's fused_dns_matvec (OpenMP, all host threads) through
    its own bench_matvec (median of `repeats` after one warmup) on a row slice
    of every GEMV of one decoder layer.  Returns (GB/s, seconds, bytes, cores, desc)."""
    from oracle.oracle import Reference, make_x
    ref = Reference()
    cores = os.cpu_count() or 1
    ref.lib.ref_set_threads(cores)
    total_s, total_b = 0.0, 0
    for (name, rows, cols), L in zip(SHAPES, host_layers):
        n = max(32, int(rows * frac))
        Ls = slice_rows(L, 0, n)
        rl = ref.layer(Ls, top_k=10)
        med, bt = rl.bench("fused", make_x(cols).astype(np.float32), repeats=repeats)
        total_s += med
        total_b += bt
    desc = (f"reference dsq::fused_dns_matvec via dsq::bench_matvec (median of {repeats} after "
            f"1 warmup, OpenMP {cores} threads) on the first {frac:.4g} of the rows of each of "
            f"the 7 GEMVs of one decoder layer ({total_b} charged bytes)")
    return total_b / total_s / 1e9, total_s, total_b, cores, desc


def cpu_model() -> str:
    """The host CPU model (lscpu 'Model name', else /proc/cpuinfo)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.strip().startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def build_host_layers(seed: int = 1234):
    from oracle.oracle import make_layer
    cache = {}
    out = []
    for name, rows, cols in SHAPES:
        key = (rows, cols)
        if key not in cache:
            cache[key] = make_layer(rows, cols, BITS, SPARSITY, seed=seed + rows + cols)
        out.append(cache[key])
    return out


def run_reference_arm(args, rank: int, world: int):
    if rank != 0:
        return
    t0 = time.time()
    host_layers = build_host_layers()
    frac = args.ref_frac
    for _ in range(args.warmup):
        cpu_reference_sample(host_layers, frac, repeats=3)
    vals, secs, byts = [], 0.0, 0
    cores, desc = 1, ""
    for _ in range(args.steps):
        v, s, b, cores, desc = cpu_reference_sample(host_layers, frac, repeats=3)
        vals.append(v)
        secs += s
        byts += b
    value = byts / secs / 1e9
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(1, "cpu"),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores,
                         "cpu_model": cpu_model(),
                         "kind": "reference", "sample": desc},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(time.time() - t0, 1),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer
    from oracle.oracle import make_x, to_quantized_layer

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    t_setup = time.time()
    host_layers = build_host_layers()
    qls = [to_quantized_layer(L, name=n) for L, (n, _, _) in zip(host_layers, SHAPES)]
    bytes_step = sum(int(N.lib.dsq_bytes_touched_estimate(r, c, BITS, 0, L.nnz))
                     for L, (_, r, c) in zip(host_layers, SHAPES))
    n_rot = args.rotation
    # n_rot decoder layers of distinct device weights
    dls = [[DeviceLayer(q, device=local_rank) for q in qls] for _ in range(n_rot)]
    info = dls[0][0].info()
    # graphs must be captured on a non-default stream; everything runs on it
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    sp = st.cuda_stream
    # activations: step input x (fp16) + 7 fp16 outputs, one set per rotation slot
    xs = [torch.from_numpy(make_x(4096, seed=100 + i).view(np.int16)).to(dev)
          for i in range(n_rot)]
    ys = [[torch.empty(r, dtype=torch.int16, device=dev) for (_, r, _) in SHAPES]
          for _ in range(n_rot)]

    def step_input(slot: int, first: bool):
        return xs[slot] if first else ys[(slot - 1) % n_rot][len(SHAPES) - 1]

    def launch_step(slot: int, first: bool = False):
        outs = ys[slot]
        for j, ((_, r, c), dl) in enumerate(zip(SHAPES, dls[slot])):
            src = step_input(slot, first) if CHAIN_IN[j] < 0 else outs[CHAIN_IN[j]]
            dl.gemv(N.KERNEL_FUSED, src.data_ptr(), N.F16, outs[j].data_ptr(), N.F16, sp)

    # eager warm-up (sets kernel attributes, first-touch)
    for s in range(max(1, args.warmup)):
        launch_step(s % n_rot, first=(s == 0))
    torch.cuda.synchronize()

    if args.mode == "graph":
        # one launch per GEMV (programmatic dependent launch), captured in a CUDA graph
        def capture(nsteps: int, offset: int):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for s in range(nsteps):
                    launch_step((offset + s) % n_rot, first=(s == 0))
            return g

        g_warm, g_time = capture(args.warmup, 0), capture(args.steps, args.warmup)
        run_warm, run_time = g_warm.replay, g_time.replay
        launches = args.steps * len(SHAPES)
        kernel_name = "sqz::stack_gemv<3> (1 layer per launch)"
    else:
        # ONE persistent launch runs all K steps (K*7 chained GEMVs)
        from paper_2306_07629_b200 import DeviceStack

        def build_stack(nsteps: int, offset: int):
            layers, deps, xp, yp = [], [], [], []
            prev_down = -1
            for s in range(nsteps):
                slot = (offset + s) % n_rot
                base = len(layers)
                for j, dl in enumerate(dls[slot]):
                    layers.append(dl)
                    if CHAIN_IN[j] < 0 and prev_down < 0:
                        deps.append(-1)
                        xp.append(xs[slot].data_ptr())
                    else:
                        deps.append(prev_down if CHAIN_IN[j] < 0 else base + CHAIN_IN[j])
                        xp.append(0)
                    yp.append(ys[slot][j].data_ptr())
                prev_down = base + len(SHAPES) - 1
            return DeviceStack(layers, deps, xp, yp, N.F16)

        s_warm, s_time = build_stack(args.warmup, 0), build_stack(args.steps, args.warmup)
        run_warm = lambda: s_warm.run(sp)  # noqa: E731
        run_time = lambda: s_time.run(sp)  # noqa: E731
        launches = 1
        kernel_name = "sqz::stack_gemv<3> (persistent, all K*7 GEMVs in one launch)"
    run_warm()
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup

    # soak: keep the GPU under load while the clock sampler runs
    sampler = ClockSampler(local_rank)
    sampler.start()
    t_end = time.time() + args.soak
    while time.time() < t_end:
        run_warm()
        torch.cuda.synchronize()
    # W untimed warm-up steps, then exactly K timed steps
    run_warm()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    run_time()
    e1.record(st)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clocks = sampler.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * bytes_step * args.steps / (ms * 1e-3) / 1e9
    us_layer = ms_step * 1e3 / len(SHAPES)

    # ---- e2e: the decode step through the public API from HOST memory: every
    # step copies its input x (pinned host fp16) to the device, runs the
    # step's 7-GEMV chain (one persistent stack launch, DeviceStack.run) and
    # reads the step's result (the down-projection output) back to pinned host
    # memory, synchronizing each step.  Layers rotate like the timed region.
    e2e = None
    if not args.no_e2e and args.mode == "stack":
        from paper_2306_07629_b200 import DeviceStack
        n_e2e = args.e2e_steps
        x_dev = torch.empty(4096, dtype=torch.int16, device=dev)
        y_host = torch.empty(SHAPES[-1][1], dtype=torch.int16).pin_memory()
        x_host = torch.from_numpy(make_x(4096, seed=7).view(np.int16)).pin_memory()
        one = []
        for slot in range(n_rot):
            layers, deps, xp, yp = [], [], [], []
            for j, dl in enumerate(dls[slot]):
                layers.append(dl)
                deps.append(-1 if CHAIN_IN[j] < 0 else CHAIN_IN[j])
                xp.append(x_dev.data_ptr() if CHAIN_IN[j] < 0 else 0)
                # the step's result (the down projection) is written by the
                # kernel straight into pinned host memory (zero-copy D2H)
                yp.append(y_host.data_ptr() if j == len(SHAPES) - 1 else ys[slot][j].data_ptr())
            one.append(DeviceStack(layers, deps, xp, yp, N.F16))

        def e2e_step(slot):
            one[slot].run_host(x_host.data_ptr(), x_dev.data_ptr(), x_host.numel() * 2,
                               None, None, 0, sp)

        for s in range(3):
            e2e_step(s % n_rot)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for s in range(n_e2e):
            e2e_step(s % n_rot)
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        launch_form = {
            "value": round(world * bytes_step * n_e2e / el / 1e9, 2), "unit": "GB/s",
            "ms_per_step": round(el / n_e2e * 1e3, 4),
            "api": "DeviceStack.run_host (dsq_cuda_stack_run_host), one launch + one stream "
                   "synchronisation per step: pinned host x read by a 1-CTA upload kernel "
                   "overlapped with the stack kernel's prologue (PDL), the step output written "
                   "straight into pinned host memory"}

        # the serving loop (dsq_cuda_serve_*): the n_e2e steps as ONE resident
        # launch fed step by step -- x_host -> x_dev on the copy engine, the
        # step's doorbell behind it, the step's result (down projection) written
        # by the kernel into pinned host memory and read into a numpy array
        # once the kernel's completion word for the step arrives
        y_srv = torch.zeros(SHAPES[-1][1], dtype=torch.int16).pin_memory()
        y_np = y_srv.numpy()
        y_out = np.empty(SHAPES[-1][1], dtype=np.int16)
        layers, deps, xp, yp, gate, notify = [], [], [], [], [], []
        for st_i in range(n_e2e):
            slot, base = st_i % n_rot, len(layers)
            for j, dl in enumerate(dls[slot]):
                last = j == len(SHAPES) - 1
                layers.append(dl)
                deps.append(-1 if CHAIN_IN[j] < 0 else base + CHAIN_IN[j])
                xp.append(x_dev.data_ptr() if CHAIN_IN[j] < 0 else 0)
                gate.append(st_i + 1 if CHAIN_IN[j] < 0 else 0)
                yp.append(ys[slot][j].data_ptr())
                notify.append(st_i + 1 if last else 0)
        served = DeviceStack(layers, deps, xp, yp, N.F16, serve_gate=gate, serve_notify=notify)
        torch.cuda.synchronize()
        y_args = (y_srv.data_ptr(), SHAPES[-1][1] * 2)
        served.serve_begin(x_dev.data_ptr(), x_host.numel() * 2, *y_args, sp)  # warm-up
        for st_i in range(3):  # (the steps not fed are released by serve_end)
            served.serve_step(x_host.data_ptr())
        served.serve_end()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        served.serve_begin(x_dev.data_ptr(), x_host.numel() * 2, *y_args, sp)
        for st_i in range(n_e2e):
            served.serve_step(x_host.data_ptr())
            np.copyto(y_out, y_np)
        served.serve_end()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        serving = {
            "value": round(world * bytes_step * n_e2e / el / 1e9, 2), "unit": "GB/s",
            "ms_per_step": round(el / n_e2e * 1e3, 4),
            "api": "DeviceStack.serve_begin/serve_step/serve_end (dsq_cuda_stack_create_served, "
                   "dsq_cuda_serve_*): the decode steps as one resident launch (inside the "
                   "timed region) fed per step from host memory -- x copied into pinned "
                   "staging + a doorbell word, CTA 0 of the kernel pulls the bytes over PCIe "
                   "into the device x and releases the grid; the last layer's finishing warps "
                   "write the step output straight into pinned host memory as tagged 64-bit "
                   "words (4 payload bytes + the step number: no fence, no gather; 2x the "
                   "payload on the wire), the host waits for every tag and copies the payload "
                   "out; no CUDA call, launch or stream synchronisation per step "
                   "(tools/serve_trace.py: ~35 us of GPU work + ~7.5 us host round trip per step)"}
        # the headline e2e is the faster of the two public per-step paths
        fast, other = (serving, launch_form) if serving["value"] >= launch_form["value"] \
            else (launch_form, serving)
        e2e = dict(fast)
        e2e.update({"h2d_bytes_per_step": 4096 * 2, "d2h_bytes_per_step": SHAPES[-1][1] * 2,
                    "steps": n_e2e,
                    ("per_step_launch" if other is launch_form else "serving_loop"): other})
        # the reference-signature host call, per GEMV (fp32 host x -> fp64 host y,
        # dsq_cuda_matvec_host = fused_dns_matvec(layer, x)), for comparison
        xh = make_x(4096).astype(np.float32)
        big = np.empty(11008, dtype=np.float32)

        def host_step(slot):
            outs = []
            for j, ((_, r, c), dl) in enumerate(zip(SHAPES, dls[slot])):
                src = xh if CHAIN_IN[j] < 0 else big[:c]
                if CHAIN_IN[j] >= 0:
                    src[:] = outs[CHAIN_IN[j]]
                outs.append(dl.matvec_host(N.KERNEL_FUSED, src).astype(np.float32))

        nh = 20
        for s in range(min(nh, n_rot)):  # every layer's host staging once
            host_step(s)
        t0 = time.perf_counter()
        for s in range(nh):
            host_step(s % n_rot)
        el = time.perf_counter() - t0
        e2e["per_gemv_host_api"] = {
            "value": round(world * bytes_step * nh / el / 1e9, 2), "unit": "GB/s",
            "ms_per_step": round(el / nh * 1e3, 3),
            "api": "dsq_cuda_matvec_host per GEMV (fp32 host x -> fp64 host y)"}

    if rank != 0:
        return
    pk = peaks()
    peak = float(pk.get("hbm_gbs", 6650.0))
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("dram_bytes_per_step")
        except Exception:
            traffic = None
    per_rank = value / world
    # the roofline model's prediction (paper_2306_07629_b200/roofline.py):
    # reference-charged bytes of the step's 7 GEMVs at the HBM peak
    from paper_2306_07629_b200 import roofline as RL
    hw = RL.b200_profile()
    pred_us = sum(RL.gemv_cost(r, c, 3, L.nnz, hw).predicted_time
                  for L, (_, r, c) in zip(host_layers, SHAPES)) * 1e6
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic (random fp16 centroids/indices/deltas; weights random-init)",
        "config": workload_config(n_rot, "tp1" if world == 1 else f"replicas{world}"),
        "us_per_layer": round(us_layer, 3),
        "decode_tok_s_linear": round(1e3 / (ms_step * LLAMA7B_LAYERS), 1),
        "frac_of_8TBs": round(per_rank / 8000.0, 4),
        "roofline": {"bound": "hbm", "achieved": round(per_rank, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(per_rank / peak, 4), "traffic": traffic,
                     "kernel": kernel_name,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else "fallback",
                     "algorithmic_bytes_per_step": bytes_step,
                     "model": {"profile": hw.name, "predicted_us_per_step": round(pred_us, 3),
                               "measured_us_per_step": round(ms_step * 1e3, 3)}},
        "e2e": e2e, "clocks": clocks, "gpu_launches": launches,
        "gemvs_timed": args.steps * len(SHAPES), "mode": args.mode,
        "schedule": {"workers": info.workers, "ctas": info.ctas},
        "setup_s": round(setup_s, 1),
    }
    if world == 1 and not args.no_per_layer:
        line["per_layer"] = per_layer_bench(dev, peak)
        line["model_stacks"] = model_stacks_bench(dev, peak)
        line["batch_sweep"] = batch_sweep_bench(dev, peak)
    if world == 1 and not args.no_cpu_baseline:
        v, s, b, cores, desc = cpu_reference_sample(host_layers, args.ref_frac, repeats=3)
        line["cpu_baseline"] = {"value": round(v, 4), "unit": "GB/s", "cores": cores,
                                "cpu_model": cpu_model(),
                                "kind": "reference", "sample": desc}
    print(json.dumps(line), flush=True)


PER_LAYER = [  # (name, rows, cols, bits, sparsity): BASELINE configs[0] and configs[1]
    ("configs0_4096x4096_4bit_dense", 4096, 4096, 4, 0.0),
    ("configs1_4096x4096_3bit_s045", 4096, 4096, 3, SPARSITY),
    ("configs1_11008x4096_3bit_s045", 11008, 4096, 3, SPARSITY),
    ("configs1_4096x11008_3bit_s045", 4096, 11008, 3, SPARSITY),
]


def per_layer_bench(dev, peak: float, launches: int = 200) -> dict:
    """µs per layer (the metric's first item) for single-layer products:
    `isolated` = one dsq_cuda_gemv launch per product (K launches back to back
    under PDL, captured in a CUDA graph so host launch cost is not timed);
    `in_stack` = the same products as independent layers of one persistent
    launch.  Weights rotate over copies totalling > 128 MB (> L2).  CUDA
    events on the launching stream."""
    import torch
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from oracle.oracle import make_layer, make_x, to_quantized_layer
    out = {}
    st = torch.cuda.current_stream(dev)
    for name, rows, cols, bits, sp in PER_LAYER:
        L = make_layer(rows, cols, bits, sp, seed=rows + cols + bits)
        q = to_quantized_layer(L, name=name)
        nbytes = int(N.lib.dsq_bytes_touched_estimate(rows, cols, bits, 0, L.nnz))
        ncopy = max(4, -(-(160 << 20) // nbytes))
        dls = [DeviceLayer(q, device=dev.index or 0) for _ in range(ncopy)]
        x = torch.from_numpy(make_x(cols).view(np.int16)).to(dev)
        ys = [torch.empty(rows, dtype=torch.int16, device=dev) for _ in range(ncopy)]

        def launch_all(k):
            for i in range(k):
                dls[i % ncopy].gemv(N.KERNEL_FUSED, x.data_ptr(), N.F16, ys[i % ncopy].data_ptr(),
                                    N.F16, st.cuda_stream)
        launch_all(ncopy)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            launch_all(launches)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        us_iso = e0.elapsed_time(e1) * 1e3 / launches
        stk = DeviceStack(dls * max(1, launches // ncopy), [-1] * (ncopy * max(1, launches // ncopy)),
                          [x.data_ptr()] * (ncopy * max(1, launches // ncopy)),
                          [y.data_ptr() for y in ys] * max(1, launches // ncopy), N.F16)
        n_in = ncopy * max(1, launches // ncopy)
        stk.run(st.cuda_stream)
        torch.cuda.synchronize()
        e0.record(st)
        stk.run(st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        us_stk = e0.elapsed_time(e1) * 1e3 / n_in
        gbs_iso, gbs_stk = nbytes / us_iso / 1e3, nbytes / us_stk / 1e3
        out[name] = {"algorithmic_bytes": nbytes, "copies_rotated": ncopy,
                     "isolated_us": round(us_iso, 3), "isolated_GBs": round(gbs_iso, 1),
                     "isolated_frac": round(gbs_iso / peak, 4),
                     "in_stack_us": round(us_stk, 3), "in_stack_GBs": round(gbs_stk, 1),
                     "in_stack_frac": round(gbs_stk / peak, 4)}
        del g, stk, dls
        torch.cuda.synchronize()
    return out


def model_stacks_bench(dev, peak: float, models=("13b", "65b"), tokens: int = 2) -> dict:
    """BASELINE configs[2] / configs[3] (N = 1): whole LLaMA-13B / 65B linear
    stacks (every decoder layer's 7 GEMVs, chained like the bench, 3-bit +
    0.45% CSR, batch 1) as ONE persistent launch per `tokens` decode steps;
    decoder layers rotate over distinct device weights totalling > 256 MB.
    CUDA events on the launching stream."""
    import torch
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from paper_2306_07629_b200.tp import decoder_chain
    from oracle.oracle import make_x, nnz_for
    out = {}
    st = torch.cuda.current_stream(dev)
    for m in models:
        h, f, n_dec = MODELS[m]
        shapes = model_shapes(m)
        cache = {}
        qls = []
        for _, r, c in shapes:
            if (r, c) not in cache:
                cache[(r, c)] = synthetic_layer(r, c, seed=r * 7 + c)
            qls.append(cache[(r, c)])
        dec_bytes = sum(int(N.lib.dsq_bytes_touched_estimate(r, c, BITS, 0,
                                                            nnz_for(r * c, SPARSITY)))
                        for _, r, c in shapes)
        rot = max(2, -(-(256 << 20) // dec_bytes))
        dls = [[DeviceLayer(q, device=dev.index or 0) for q in qls] for _ in range(rot)]
        x = torch.from_numpy(make_x(h).view(np.int16)).to(dev)
        ys = [[torch.empty(q.rows, dtype=torch.int16, device=dev) for q in qls] for _ in range(rot)]
        deps, _, _ = decoder_chain(tokens * n_dec, 1)
        layers, yp = [], []
        for t in range(tokens * n_dec):
            layers += dls[t % rot]
            yp += [y.data_ptr() for y in ys[t % rot]]
        stk = DeviceStack(layers, deps, [x.data_ptr() if d < 0 else 0 for d in deps], yp, N.F16)
        stk.run(st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        stk.run(st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        gbs = dec_bytes * n_dec * tokens / (ms * 1e-3) / 1e9
        out[f"llama{m}"] = {
            "config": "BASELINE configs[2]" if m == "13b" else "BASELINE configs[3] (1 GPU)",
            "decoder_layers": n_dec, "tokens": tokens, "ms_per_token": round(ms / tokens, 4),
            "decode_tok_s_linear": round(tokens / (ms * 1e-3), 1),
            "us_per_gemv": round(ms * 1e3 / (tokens * n_dec * 7), 3),
            "GBs": round(gbs, 1), "frac": round(gbs / peak, 4), "rotation": rot,
            "bytes_per_token": dec_bytes * n_dec}
        del stk, dls
        torch.cuda.synchronize()
    return out


def batch_sweep_bench(dev, peak: float, reps: int = 50) -> list:
    """BASELINE configs[4] (a bounded slice): LLaMA-7B shapes, 3-bit + 0.45%,
    batch 1/2/4/8/16, one fused product per batch (K7 with 2..4 vectors
    sharing each decoded fragment, K11 + its finish kernel beyond); bytes =
    weights once + the B
    x / y vectors; layers rotate over > 256 MB."""
    import torch
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer
    from oracle.oracle import make_layer, make_x, to_quantized_layer
    st = torch.cuda.current_stream(dev).cuda_stream
    out = []
    for rows, cols in [(4096, 4096), (11008, 4096)]:
        L = make_layer(rows, cols, BITS, SPARSITY, seed=3)
        q = to_quantized_layer(L)
        wbytes = int(N.lib.dsq_bytes_touched_estimate(rows, cols, BITS, 0, L.nnz))
        nl = max(2, -(-(256 << 20) // wbytes))
        dls = [DeviceLayer(q, device=dev.index or 0) for _ in range(nl)]
        base = None
        for B in (1, 2, 4, 8, 16):
            x = torch.from_numpy(np.stack([make_x(cols, seed=b) for b in range(B)])
                                 .view(np.int16)).to(dev)
            y = torch.empty(B, rows, dtype=torch.float16, device=dev)
            for i in range(nl):
                N.check(N.lib.dsq_cuda_gemv(dls[i].handle, N.KERNEL_FUSED, x.data_ptr(), N.F16,
                                            y.data_ptr(), N.F16, B, st))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(reps):
                N.check(N.lib.dsq_cuda_gemv(dls[i % nl].handle, N.KERNEL_FUSED, x.data_ptr(),
                                            N.F16, y.data_ptr(), N.F16, B, st))
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            gbs = (wbytes + (B - 1) * (rows + cols) * 2) / us / 1e3
            base = base or us
            out.append({"shape": f"{rows}x{cols}", "batch": B, "us": round(us, 3),
                        "GBs": round(gbs, 1), "frac": round(gbs / peak, 4),
                        "speedup_vs_B_x_batch1": round(B * base / us, 2)})
        del dls
        torch.cuda.synchronize()
    return out


class TPUnavailable(RuntimeError):
    pass


MODELS = {"7b": (4096, 11008, 32), "13b": (5120, 13824, 40),
          "65b": (8192, 22016, 80)}  # hidden, ffn, decoder layers


def model_shapes(model: str):
    h, f, _ = MODELS[model]
    return [("v", h, h), ("q", h, h), ("o", h, h), ("k", h, h), ("up", f, h), ("gate", f, h),
            ("down", h, f)]


def synthetic_layer(rows, cols, seed, bits=BITS, sparsity=SPARSITY):
    """A QuantizedLayer generated directly in the reference packed layout
    (uniform 3-bit indices = uniform payload bytes; outlier positions cleared
    to index 0 as quantize_layer does, pipeline.cpp:25-32), so 65B shapes
    build in seconds (bench setup only)."""
    from paper_2306_07629_b200 import CsrMatrix, PackedDense, QuantizedLayer
    from oracle.oracle import nnz_for
    rng = np.random.default_rng(seed)
    stride = (cols * bits + 7) // 8
    payload = rng.integers(0, 256, size=rows * stride, dtype=np.uint8)
    luts = np.sort(rng.normal(0.0, 0.02, size=(rows, 1 << bits)).astype(np.float16),
                   axis=1).reshape(-1)
    pos = np.unique(rng.integers(0, rows * cols, size=nnz_for(rows * cols, sparsity),
                                 dtype=np.int64))
    r, c = pos // cols, pos % cols
    for b in range(bits):
        bp = r * stride * 8 + c * bits + b
        np.bitwise_and.at(payload, bp >> 3, np.uint8(0xff) ^ (np.uint8(1) << (bp & 7).astype(np.uint8)))
    row_ptr = np.zeros(rows + 1, np.uint32)
    np.add.at(row_ptr, r + 1, 1)
    row_ptr = np.cumsum(row_ptr, dtype=np.uint64).astype(np.uint32)
    vals = rng.normal(0.0, 0.2, size=pos.size).astype(np.float16)
    return QuantizedLayer(f"{rows}x{cols}", rows, cols, PackedDense(bits, rows, cols, luts, payload),
                          CsrMatrix(rows, cols, row_ptr, c.astype(np.uint16), vals), 10)


def run_ours_tp(args, rank: int, world: int, local_rank: int):
    """A decoder-layer chain of `--workload` shapes (65B by default at N > 1:
    BASELINE configs[3]) tensor-parallel over the N GPUs (Megatron split:
    v,q,k,up,gate column-parallel, o,down row-parallel, tp.py), the two
    all-reduces per decoder layer fused into the persistent stack kernel over
    NVLink peer memory (CUDA IPC-mapped receive buffers).  Each rank generates
    its own shards of the layer shapes directly (synthetic weights).  value =
    the whole decoder layer's reference-charged bytes per step / step time,
    max over ranks (strong scaling: the model is fixed, N GPUs share it)."""
    import torch
    import torch.distributed as dist
    import paper_2306_07629_b200._native as N
    from paper_2306_07629_b200 import DeviceLayer, DeviceStack
    from paper_2306_07629_b200.dsq import TPContext
    from paper_2306_07629_b200.tp import ROW_PARALLEL, decoder_chain, split_range
    from oracle.oracle import make_x, nnz_for

    model = args.workload if args.workload != "auto" else "65b"
    h, f, n_dec = MODELS[model]
    shapes = model_shapes(model)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    t_setup = time.time()
    bytes_step = sum(int(N.lib.dsq_bytes_touched_estimate(r, c, BITS, 0,
                                                          nnz_for(r * c, SPARSITY)))
                     for _, r, c in shapes)
    # this rank's shard shapes (32-aligned splits, tp.shard_decoder's)
    shard_shapes = []
    for name, r, c in shapes:
        if world == 1:
            shard_shapes.append((r, c))
        elif name in ROW_PARALLEL:
            c0, c1 = split_range(c, world, rank, 32)
            shard_shapes.append((r, c1 - c0))
        else:
            r0, r1 = split_range(r, world, rank, 32)
            shard_shapes.append((r1 - r0, c))
    cache = {}
    shards = []
    for i, (r, c) in enumerate(shard_shapes):
        if (r, c) not in cache:
            cache[(r, c)] = synthetic_layer(r, c, seed=1000 * rank + r * 7 + c)
        shards.append(cache[(r, c)])
    shard_bytes = sum(int(N.lib.dsq_bytes_touched_estimate(q.rows, q.cols, BITS, 0,
                                                           q.sparse.nnz())) for q in shards)
    # rotation: distinct device weights per step totalling > 2x L2 per GPU
    n_rot = max(2, -(-(256 << 20) // shard_bytes)) if args.rotation_auto else args.rotation
    if world > 1:  # every rank must run the same launch sequence
        t = torch.tensor([n_rot], device=dev, dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        n_rot = int(t.item())
    dls = [[DeviceLayer(q, device=local_rank) for q in shards] for _ in range(n_rot)]
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    ctx = None
    if world > 1:
        ctx = TPContext(world, rank, max_rows=h, max_grid=sms, device=local_rank)
        handles = [None] * world
        dist.all_gather_object(handles, ctx.ipc_handle)
        ok = 1
        try:
            ctx.connect(handles)
        except Exception as e:
            print(f"rank {rank}: tp connect failed: {e}", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not int(flag.item()):
            raise TPUnavailable("CUDA IPC peer mapping failed")
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    sp = st.cuda_stream
    x = torch.from_numpy(make_x(h, seed=100).view(np.int16)).to(dev)
    ys = [[torch.empty(q.rows, dtype=torch.int16, device=dev) for q in shards]
          for _ in range(n_rot)]

    def build(nsteps, offset):
        deps, reduce, _ = decoder_chain(nsteps, 1)
        layers, yp = [], []
        for s_ in range(nsteps):
            slot = (offset + s_) % n_rot
            layers += dls[slot]
            yp += [y.data_ptr() for y in ys[slot]]
        xp = [x.data_ptr() if d < 0 else 0 for d in deps]
        if ctx is None:
            return DeviceStack(layers, deps, xp, yp, N.F16)
        return DeviceStack(layers, deps, xp, yp, N.F16, reduce=reduce, tp=ctx)

    s_warm, s_time = build(args.warmup, 0), build(args.steps, args.warmup)
    # every rank runs the same launch sequence (the reduce tags advance per
    # launch): fixed counts, no time-based loops
    for _ in range(2):
        s_warm.run(sp)
    torch.cuda.synchronize()
    if ctx is not None:
        # validate the fused reduce before timing: no watchdog event and the
        # same reduced outputs (the last step's o and down) on every rank
        ok = 1
        try:
            ctx.check()
        except Exception as e:
            print(f"rank {rank}: tp watchdog: {e}", file=sys.stderr)
            ok = 0
        slot = (args.warmup - 1) % n_rot
        sig = torch.stack([ys[slot][2].to(torch.int64).sum(), ys[slot][6].to(torch.int64).sum()])
        sigs = [torch.zeros_like(sig) for _ in range(world)]
        dist.all_gather(sigs, sig)
        if any(not torch.equal(g, sigs[0]) for g in sigs):
            ok = 0
        flag = torch.tensor([ok], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not int(flag.item()):
            raise TPUnavailable("fused TP reduce failed validation (watchdog or rank mismatch)")
    setup_s = time.time() - t_setup
    sampler = ClockSampler(local_rank)
    sampler.start()
    t0 = time.time()
    s_warm.run(sp)
    torch.cuda.synchronize()
    per_run = max(time.time() - t0, 1e-5)
    n_soak = torch.tensor([int(args.soak / per_run) + 1], device=dev, dtype=torch.int64)
    if world > 1:
        dist.all_reduce(n_soak, op=dist.ReduceOp.MAX)
    for i in range(int(n_soak.item())):
        s_warm.run(sp)
        if i % 64 == 63:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    s_warm.run(sp)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s_time.run(sp)
    e1.record(st)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clocks = sampler.stop()
    if ctx is not None:
        ctx.check()
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    value = bytes_step * args.steps / (ms * 1e-3) / 1e9

    # e2e: one-step stacks from host memory (x H2D, the step's reduced down
    # output D2H) through DeviceStack.run on every rank
    e2e = None
    if not args.no_e2e:
        one = [build(1, slot) for slot in range(n_rot)]
        x_host = torch.from_numpy(make_x(h, seed=7).view(np.int16)).pin_memory()
        y_host = torch.empty(shards[-1].rows, dtype=torch.int16).pin_memory()

        def step(slot):
            x.copy_(x_host, non_blocking=True)
            one[slot].run(sp)
            y_host.copy_(ys[slot][-1], non_blocking=True)
            st.synchronize()

        for s_ in range(3):
            step(s_ % n_rot)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for s_ in range(args.e2e_steps):
            step(s_ % n_rot)
        el = time.perf_counter() - t0
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
        if ctx is not None:
            ctx.check()
        e2e = {"value": round(bytes_step * args.e2e_steps / el / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": h * 2, "d2h_bytes_per_step": shards[-1].rows * 2,
               "steps": args.e2e_steps, "ms_per_step": round(el / args.e2e_steps * 1e3, 4),
               "api": "DeviceStack.run (dsq_cuda_stack_create_tp) per decoder-layer step on "
                      "every rank: pinned host x -> device, the step's reduced output -> host"}
    if rank != 0:
        return
    pk = peaks()
    peak = float(pk.get("hbm_gbs", 6650.0))
    per_gpu = value / world
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic (random fp16 centroids/indices/deltas per rank shard; "
                "weights random-init)",
        "config": {
            "workload": f"llama{model[:-1]}-decoder-linear-chain tensor-parallel: q,k,v,o "
                        f"{h}x{h}; gate,up {f}x{h}; down {h}x{f}; 3-bit LUT + 0.45% CSR; batch 1 "
                        f"(BASELINE configs[3] for 65b)",
            "gemvs_per_step": 7, "bits": BITS, "sparsity": SPARSITY, "batch": 1,
            "l2": f"inputs larger than L2: rotation over {n_rot} decoder layers of distinct "
                  f"device weights ({shard_bytes * n_rot / 2**20:.0f} MiB per GPU)",
            "parallelism": f"tp{world} (v,q,k,up,gate column-parallel; o,down row-parallel; "
                           f"all-reduce fused into the stack kernel over NVLink peer memory)"
            if world > 1 else "tp1"},
        "us_per_layer": round(ms_step * 1e3 / 7, 3),
        "decode_tok_s_linear": round(1e3 / (ms_step * n_dec), 1),
        "frac_of_8TBs": round(per_gpu / 8000.0, 4),
        "roofline": {"bound": "hbm", "achieved": round(per_gpu, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(per_gpu / peak, 4), "traffic": None,
                     "kernel": "sqz::stack_gemv<3> (persistent" +
                               (", fused TP reduce)" if world > 1 else ")"),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else "fallback",
                     "algorithmic_bytes_per_step": bytes_step, "per": "GPU",
                     "per_gpu_shard_bytes_per_step": shard_bytes},
        "e2e": e2e, "clocks": clocks, "gpu_launches": 1, "gemvs_timed": args.steps * 7,
        "mode": "stack-tp", "setup_s": round(setup_s, 1),
    }
    if world > 1 and model == "65b":
        # `bench.py --gpus 1` measures BASELINE configs[1] (the 7B chain); the
        # same 65B chain on one GPU (`--workload 65b`), for a same-workload
        # scaling read, is the builder's committed measurement
        ref1 = ROOT / "profiles" / "r02_bench_65b_tp1.json"
        if ref1.exists():
            try:
                v1 = json.loads(ref1.read_text())["value"]
                line["same_workload_1gpu"] = {
                    "value": v1, "unit": "GB/s", "source": str(ref1.relative_to(ROOT)),
                    "note": "python bench.py --workload 65b at N = 1 (not this run)"}
            except Exception:
                pass
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["stack", "graph"], default="stack",
                    help="stack: one persistent launch for all K steps; graph: one launch "
                         "per GEMV captured in a CUDA graph")
    ap.add_argument("--rotation", type=int, default=16,
                    help="decoder layers of distinct device weights (working set >> L2; the "
                         "TP path sizes its own rotation unless --no-rotation-auto)")
    ap.add_argument("--no-rotation-auto", dest="rotation_auto", action="store_false")
    ap.add_argument("--soak", type=float, default=1.0, help="seconds of load before timing")
    ap.add_argument("--workload", choices=["auto", "7b", "13b", "65b"], default="auto",
                    help="auto: the LLaMA-7B chain (configs[1]) at N=1, the 65B chain "
                         "tensor-parallel (configs[3]) at N>1")
    ap.add_argument("--multi", choices=["tp", "replicas"], default="tp",
                    help="N>1: tensor-parallel decoder layers (fused all-reduce) or N replicas")
    ap.add_argument("--force-tp", action="store_true",
                    help="dev: run the TP path even at N=1 (under torchrun)")
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-layer", action="store_true",
                    help="skip the per-layer (configs[0]/[1]), model-stack (configs[2]/[3] at "
                         "N=1) and batch-sweep (configs[4]) sections")
    ap.add_argument("--ref-frac", type=float, default=1 / 16,
                    help="row fraction of each GEMV in the CPU sample")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    use_tp = (world > 1 and args.multi == "tp") or args.force_tp or args.workload == "65b"
    if world > 1 or args.force_tp:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if use_tp:
            # a TP failure is an error (exit non-zero), never a silent switch to
            # replicas: --multi replicas asks for replicas explicitly
            run_ours_tp(args, rank, world, local_rank)
            return
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1 or args.force_tp:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
