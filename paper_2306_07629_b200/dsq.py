"""Python mirror of the reference ``dsq`` hot-path interface, backed by sm_100a.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/dsq/{packfmt,dns,kernels}.hpp, so parity tests
read like the reference's own tests:

  PackedDense        packfmt.hpp:16-33   (luts fp32 or fp16, payload LSB-first)
  CsrMatrix          dns.hpp:14-24       (values = deltas vs lut_row[0])
  QuantizedLayer     packfmt.hpp:50-61
  lut_matvec         kernels.hpp:20      -> DSQ_KERNEL_LUT
  csr_matvec         kernels.hpp:24      -> DSQ_KERNEL_CSR
  fused_dns_matvec   kernels.hpp:31      -> DSQ_KERNEL_FUSED
  dense_matvec       kernels.hpp:35      -> K4 fp16 dense GEMV
  bench_matvec       kernels.hpp:74      (median of >= 3 after one warmup)
  bytes_touched_estimate kernels.hpp:79

Every product runs on the GPU through ``libdsq_cuda.so``; the host-vector
entry points (returning float64 like the reference's std::vector<double>)
go through ``dsq_cuda_matvec_host`` (H2D x, launch, D2H y).  The ``exec``
argument accepts the reference's ``Exec`` values and ``Exec.cuda``; all of
them execute on the device (the reference's serial/parallel distinction is a
CPU threading choice with bit-identical results, kernels.hpp:13-16).
"""
from __future__ import annotations

import ctypes as C
import enum
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import DsqError, check, lib


class Exec(enum.Enum):  # kernels.hpp:17 + the device
    serial = 0
    parallel = 1
    cuda = 2


class BenchKernel(enum.IntEnum):  # kernels.hpp:71
    lut = N.KERNEL_LUT
    csr = N.KERNEL_CSR
    fused = N.KERNEL_FUSED
    reference = N.KERNEL_REFERENCE


def row_stride(cols: int, bits: int) -> int:
    return (cols * bits + 7) // 8  # packfmt.hpp:26


@dataclass
class PackedDense:
    bits: int
    rows: int
    cols: int
    luts: np.ndarray            # float32 or float16, rows*groups*2^bits
    payload: np.ndarray         # uint8, rows*row_stride
    groups_per_row: int = 1

    def levels(self) -> int:
        return 1 << self.bits

    def row_stride(self) -> int:
        return row_stride(self.cols, self.bits)


@dataclass
class CsrMatrix:
    rows: int
    cols: int
    row_ptr: np.ndarray         # uint32 rows+1
    col_idx: np.ndarray         # uint16 nnz
    values: np.ndarray          # float32 or float16 nnz

    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if len(self.row_ptr) else 0


@dataclass
class QuantizedLayer:
    name: str
    rows: int
    cols: int
    packed: PackedDense
    sparse: CsrMatrix
    hybrid_top_k: int = 0
    _device: dict = field(default_factory=dict, repr=False, compare=False)


def _ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


def layer_view(layer: QuantizedLayer, keep: list) -> N.LayerView:
    """The C-ABI view (dsq_layer_view) of a layer; the arrays it points into
    are appended to `keep` and must outlive the view."""
    p, s = layer.packed, layer.sparse

    def hold(a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        keep.append(a)
        return a

    luts = hold(p.luts, p.luts.dtype if p.luts.dtype in (np.float16, np.float32) else np.float32)
    payload = hold(p.payload, np.uint8)
    row_ptr = hold(s.row_ptr, np.uint32)
    col_idx = hold(s.col_idx, np.uint16)
    vals = hold(s.values, s.values.dtype if s.values.dtype in (np.float16, np.float32) else np.float32)
    v = N.LayerView()
    name = layer.name.encode()
    keep.append(name)
    v.name = name
    v.rows, v.cols = layer.rows, layer.cols
    v.packed.bits, v.packed.rows, v.packed.cols = p.bits, p.rows, p.cols
    v.packed.groups_per_row = p.groups_per_row
    if luts.dtype == np.float16:
        v.packed.luts_f16 = _ptr(luts)
    else:
        v.packed.luts_f32 = _ptr(luts)
    v.packed.payload = _ptr(payload)
    v.packed.payload_len = payload.size
    v.sparse.rows, v.sparse.cols, v.sparse.nnz = s.rows, s.cols, s.nnz()
    v.sparse.row_ptr = _ptr(row_ptr)
    v.sparse.col_idx = _ptr(col_idx) if col_idx.size else None
    if vals.size:
        if vals.dtype == np.float16:
            v.sparse.values_f16 = _ptr(vals)
        else:
            v.sparse.values_f32 = _ptr(vals)
    v.hybrid_top_k = layer.hybrid_top_k
    return v


class DeviceLayer:
    """Owning handle of an uploaded layer (dsq_cuda_layer_create)."""

    def __init__(self, layer: QuantizedLayer, device: int = 0):
        self._keep = []
        v = layer_view(layer, self._keep)
        h = C.c_void_p()
        check(lib.dsq_cuda_layer_create(C.byref(v), device, C.byref(h)))
        self._keep = None
        self.handle = h
        self.rows, self.cols = layer.rows, layer.cols
        self._fin = weakref.finalize(self, lib.dsq_cuda_layer_destroy, h)

    def info(self) -> N.LayerInfo:
        i = N.LayerInfo()
        check(lib.dsq_cuda_layer_get_info(self.handle, C.byref(i)))
        return i

    # -- device-buffer products (pointers: ints; stream: cudaStream_t as int)
    def gemv(self, kernel: int, x_ptr: int, x_dtype: int, y_ptr: int, y_dtype: int,
             stream: int = 0) -> None:
        check(lib.dsq_cuda_gemv(self.handle, kernel, x_ptr, x_dtype, y_ptr, y_dtype, 1, stream))

    def unpack(self, out_ptr: int, stream: int = 0) -> None:
        check(lib.dsq_cuda_unpack(self.handle, out_ptr, stream))

    def dequant(self, out_ptr: int, out_dtype: int, stream: int = 0) -> None:
        check(lib.dsq_cuda_dequant(self.handle, out_ptr, out_dtype, stream))

    def dump_frags(self, out_ptr: int, stream: int = 0) -> None:
        """fp16 A fragments of the hot decode, scattered to rows x cols (parity)."""
        check(lib.dsq_cuda_dump_frags(self.handle, out_ptr, stream))

    # -- host-vector product (the reference's signature)
    def matvec_host(self, kernel: int, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        if x.size != self.cols:
            raise DsqError(9, "dimension mismatch")
        y = np.empty(self.rows, dtype=np.float64)
        check(lib.dsq_cuda_matvec_host(self.handle, kernel, _ptr(x), _ptr(y)))
        return y

    def close(self) -> None:
        self._fin()

    @classmethod
    def _borrowed(cls, handle: C.c_void_p, owner) -> "DeviceLayer":
        """A view of a layer owned by a DeviceContainer (no finalizer)."""
        d = cls.__new__(cls)
        d.handle = handle
        d._owner = owner
        i = d.info()
        d.rows, d.cols = i.rows, i.cols
        d._fin = lambda: None
        return d


def _meta_dict(m: N.ContainerMeta) -> dict:
    return {k: getattr(m, k) for k, _ in N.ContainerMeta._fields_}


def check_container(path) -> dict:
    """load_container's checks (reference container.cpp:181-223) on the host:
    returns the QuantConfig meta or raises DsqError with the reference errc."""
    m = N.ContainerMeta()
    check(lib.dsq_container_check(str(path).encode(), C.byref(m)))
    return _meta_dict(m)


class DeviceContainer:
    """A "DSQCONT1" quantized-model container (reference container.hpp) loaded
    and uploaded: ``layers`` are device layers in file order, ``names`` their
    names, ``meta`` the QuantConfig (dsq_cuda_container_open)."""

    def __init__(self, path, device: int = 0):
        h = C.c_void_p()
        check(lib.dsq_cuda_container_open(str(path).encode(), device, C.byref(h)))
        self.handle = h
        self._fin = weakref.finalize(self, lib.dsq_cuda_container_close, h)
        m = N.ContainerMeta()
        check(lib.dsq_cuda_container_meta(h, C.byref(m)))
        self.meta = _meta_dict(m)
        n = m.n_layers
        self.layers = [DeviceLayer._borrowed(C.c_void_p(lib.dsq_cuda_container_layer(h, i)), self)
                       for i in range(n)]
        self.names = [lib.dsq_cuda_container_layer_name(h, i).decode() for i in range(n)]

    def close(self) -> None:
        self._fin()


def load_container(path, device: int = 0) -> DeviceContainer:
    return DeviceContainer(path, device)


class TPContext:
    """One rank's tensor-parallel context (dsq_cuda_tp_create): receive buffer
    + per-CTA flags for the fused all-reduce.  ``ipc_handle`` (64 bytes) goes
    to the peers; ``connect(handles)`` maps theirs (all ranks, rank order)."""

    def __init__(self, world: int, rank: int, max_rows: int, max_grid: int = 1024,
                 device: int = 0):
        h = C.c_void_p()
        self._ipc = C.create_string_buffer(64)
        check(lib.dsq_cuda_tp_create(device, world, rank, max_rows, max_grid, C.byref(h),
                                     self._ipc))
        self.handle, self.world, self.rank = h, world, rank
        self.ipc_handle = bytes(self._ipc.raw)
        self._fin = weakref.finalize(self, lib.dsq_cuda_tp_destroy, h)

    def connect(self, handles: list) -> None:
        blob = b"".join(handles)
        check(lib.dsq_cuda_tp_connect(self.handle, blob))

    def check(self) -> None:
        """Raise if a fused reduce's watchdog fired (a peer never arrived)."""
        check(lib.dsq_cuda_tp_error(self.handle))

    @staticmethod
    def connect_local(ctxs: list) -> None:
        arr = (C.c_void_p * len(ctxs))(*[c.handle.value for c in ctxs])
        check(lib.dsq_cuda_tp_connect_local(arr, len(ctxs)))


class DeviceStack:
    """A dependency chain of uploaded layers run by ONE persistent launch
    (dsq_cuda_stack_create/run).  deps[i] = index of the layer whose output
    is layer i's x, or -1 for the external fp16 buffer xs[i] (device pointer).
    With ``tp`` (a TPContext), layers with reduce[i] produce partial sums that
    the kernel all-reduces over the ranks' peer memory (dsq_cuda_stack_create_tp);
    ``grid`` = CTAs (0: one per SM).  ``batch`` (1..16) activation vectors at
    once: vector v of an external x at xs[i] + v * x_stride halves, of every
    output at ys[i] + v * y_stride elements (dsq_cuda_stack_create_batch).
    Batches the persistent kernel cannot hold run in the sequential form (one
    batched product launch per layer): see ``persistent`` / ``launches``."""

    def __init__(self, layers: list, deps: list, xs: list, ys: list, y_dtype: int,
                 reduce: list | None = None, tp: "TPContext | None" = None, grid: int = 0,
                 batch: int = 1, x_stride: int = 0, y_stride: int = 0,
                 serve_gate: list | None = None, serve_notify: list | None = None):
        n = len(layers)
        self._layers = list(layers)  # keep the layer handles alive
        self._tp = tp
        arr_l = (C.c_void_p * n)(*[d.handle.value for d in layers])
        arr_d = (C.c_int32 * n)(*deps)
        arr_x = (C.c_void_p * n)(*[x or 0 for x in xs])
        arr_y = (C.c_void_p * n)(*ys)
        h = C.c_void_p()
        if serve_gate is not None or serve_notify is not None:
            g = (C.c_uint32 * n)(*(serve_gate or [0] * n))
            nt = (C.c_uint32 * n)(*(serve_notify or [0] * n))
            check(lib.dsq_cuda_stack_create_served(arr_l, n, arr_d, arr_x, arr_y, y_dtype, g, nt,
                                                   C.byref(h)))
        elif batch > 1:
            if tp is not None or reduce is not None:
                raise DsqError(102, "batched stacks are single-GPU")
            check(lib.dsq_cuda_stack_create_batch(arr_l, n, arr_d, arr_x, arr_y, y_dtype, batch,
                                                  x_stride, y_stride, C.byref(h)))
        elif tp is None and reduce is None and grid == 0:
            check(lib.dsq_cuda_stack_create(arr_l, n, arr_d, arr_x, arr_y, y_dtype, C.byref(h)))
        else:
            red = (C.c_uint8 * n)(*([1 if r else 0 for r in reduce] if reduce else [0] * n))
            check(lib.dsq_cuda_stack_create_tp(arr_l, n, arr_d, arr_x, arr_y, y_dtype, red,
                                               tp.handle if tp is not None else None, grid,
                                               C.byref(h)))
        self.handle = h
        self._fin = weakref.finalize(self, lib.dsq_cuda_stack_destroy, h)

    def run(self, stream: int = 0) -> None:
        check(lib.dsq_cuda_stack_run(self.handle, stream))

    # serving loop (served stacks): one resident launch fed step by step
    def serve_begin(self, x_dev: int, x_bytes: int, y_host: int = 0, y_bytes: int = 0,
                    stream: int = 0) -> None:
        """Launch; every step's x_bytes of input go to x_dev (the gated layers' x),
        each step's output (notify layer, first y_bytes) to pinned y_host."""
        check(lib.dsq_cuda_serve_begin(self.handle, x_dev, x_bytes, y_host or None, y_bytes,
                                       stream))

    def serve_step(self, x_host: int) -> None:
        """Feed the next step's input (host pointer) and wait for its outputs."""
        check(lib.dsq_cuda_serve_step(self.handle, x_host))

    def serve_end(self) -> None:
        check(lib.dsq_cuda_serve_end(self.handle))

    def _info(self) -> tuple[int, int]:
        p, n = C.c_uint32(), C.c_uint32()
        check(lib.dsq_cuda_stack_info(self.handle, C.byref(p), C.byref(n)))
        return p.value, n.value

    @property
    def persistent(self) -> bool:
        """True when the whole stack is one persistent launch."""
        return bool(self._info()[0])

    @property
    def launches(self) -> int:
        """Kernel launches of the last run (1 for the persistent form)."""
        return self._info()[1]

    def run_host(self, x_host: int, x_dev: int, x_bytes: int, y_dev: int, y_host: int,
                 y_bytes: int, stream: int = 0) -> None:
        """One step from host buffers (pointers): x_host -> x_dev, run, y_dev ->
        y_host, synchronised (dsq_cuda_stack_run_host)."""
        check(lib.dsq_cuda_stack_run_host(self.handle, x_host, x_dev, x_bytes, y_dev, y_host,
                                          y_bytes, stream))


def device_layer(layer: QuantizedLayer, device: int = 0) -> DeviceLayer:
    """Upload once and cache on the layer object (layers are immutable)."""
    d = layer._device.get(device)
    if d is None:
        d = DeviceLayer(layer, device)
        layer._device[device] = d
    return d


def _as_layer_from_packed(packed: PackedDense) -> QuantizedLayer:
    empty = CsrMatrix(packed.rows, packed.cols, np.zeros(packed.rows + 1, np.uint32),
                      np.zeros(0, np.uint16), np.zeros(0, np.float32))
    return QuantizedLayer("packed", packed.rows, packed.cols, packed, empty)


def _check_x(x, cols: int, what: str) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    if x.size != cols:
        raise DsqError(9, f"{what}: dimension mismatch")  # kernels.cpp:53,71,111
    return x


def lut_matvec(packed: PackedDense, x, exec: Exec = Exec.cuda) -> np.ndarray:
    """kernels.hpp:20 -- out[r] = sum_c lut_r[idx(r,c)] * x[c]."""
    x = _check_x(x, packed.cols, "lut_matvec")
    layer = packed.__dict__.get("_layer_cache")
    if layer is None:
        layer = _as_layer_from_packed(packed)
        packed.__dict__["_layer_cache"] = layer
    return device_layer(layer).matvec_host(N.KERNEL_LUT, x)


def csr_matvec(sparse, x, exec: Exec = Exec.cuda) -> np.ndarray:
    """kernels.hpp:24 -- standard CSR product.  Accepts a CsrMatrix (like the
    reference) or a QuantizedLayer (uses its ``sparse`` part)."""
    if isinstance(sparse, QuantizedLayer):
        layer = sparse
    else:
        layer = sparse.__dict__.get("_layer_cache")
        if layer is None:
            # a CSR-only device layer: the dense part is never read by K2
            packed = PackedDense(1, sparse.rows, sparse.cols,
                                 np.zeros(sparse.rows * 2, np.float16),
                                 np.zeros(sparse.rows * row_stride(sparse.cols, 1), np.uint8))
            layer = QuantizedLayer("csr", sparse.rows, sparse.cols, packed, sparse)
            sparse.__dict__["_layer_cache"] = layer
    x = _check_x(x, layer.cols, "csr_matvec")
    return device_layer(layer).matvec_host(N.KERNEL_CSR, x)


def fused_dns_matvec(layer: QuantizedLayer, x, exec: Exec = Exec.cuda) -> np.ndarray:
    """kernels.hpp:31 -- LUT product plus the CSR deltas, one device launch."""
    x = _check_x(x, layer.cols, "fused_dns_matvec")
    return device_layer(layer).matvec_host(N.KERNEL_FUSED, x)


def dense_matvec(m, rows: int, cols: int, x, exec: Exec = Exec.cuda) -> np.ndarray:
    """kernels.hpp:35 -- plain dense product of an fp32 matrix (fp64
    accumulation of the exact fp32 products, dsq_cuda_dense_matvec_host)."""
    m = np.ascontiguousarray(m, dtype=np.float32).reshape(-1)
    if m.size != rows * cols:
        raise DsqError(9, "dense_matvec: dimension mismatch")
    x = np.ascontiguousarray(_check_x(x, cols, "dense_matvec"))
    y = np.empty(rows, dtype=np.float64)
    check(lib.dsq_cuda_dense_matvec_host(_ptr(m), rows, cols, _ptr(x), _ptr(y), 0))
    return y


def dequantize_layer(layer: QuantizedLayer) -> np.ndarray:
    """pipeline.cpp:49-75 -- the represented fp32 matrix [rows, cols]: LUT
    values, and lut_row[0] + delta (one fp32 addition) at every CSR position."""
    w = np.empty(layer.rows * layer.cols, dtype=np.float32)
    check(lib.dsq_cuda_dequantize_layer_host(device_layer(layer).handle, _ptr(w)))
    return w.reshape(layer.rows, layer.cols)


def bytes_touched_estimate(layer: QuantizedLayer) -> int:
    """kernels.cpp:205-212."""
    g = layer.packed.groups_per_row
    return int(lib.dsq_bytes_touched_estimate(layer.rows, layer.cols, layer.packed.bits,
                                              0 if g == 1 else layer.cols // g,
                                              layer.sparse.nnz()))


@dataclass
class BenchRecord:  # kernels.hpp:63-69
    kernel: str
    repeats: int
    median_seconds: float
    all_seconds: list
    bytes_touched: int


def bench_matvec(layer: QuantizedLayer, x, repeats: int, kernel: BenchKernel,
                 exec: Exec = Exec.cuda) -> BenchRecord:
    """kernels.cpp:214-282 semantics (repeats >= 3, one warmup, median), timing
    the reference-facing host call (H2D x + launch + D2H y)."""
    if repeats < 3:
        raise DsqError(11, "bench: repeats must be >= 3")
    x = _check_x(x, layer.cols, "bench")
    d = device_layer(layer)
    d.matvec_host(int(kernel), x)
    ts = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        d.matvec_host(int(kernel), x)
        ts.append(time.perf_counter() - t0)
    s = sorted(ts)
    med = s[repeats // 2] if repeats % 2 else 0.5 * (s[repeats // 2 - 1] + s[repeats // 2])
    g = layer.packed.groups_per_row
    gs = 0 if g == 1 else layer.cols // g
    rows, cols, bits, nnz = layer.rows, layer.cols, layer.packed.bits, layer.sparse.nnz()
    if kernel == BenchKernel.lut:
        bt = int(lib.dsq_bytes_touched_estimate(rows, cols, bits, gs, 0))
    elif kernel == BenchKernel.csr:
        bt = nnz * 4 + (rows + 1) * 4 + cols * 2 + rows * 2
    elif kernel == BenchKernel.fused:
        bt = bytes_touched_estimate(layer)
    else:
        bt = rows * cols * 2 + cols * 2 + rows * 2
    return BenchRecord(kernel.name, repeats, med, ts, bt)
