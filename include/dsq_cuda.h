/*
 * dsq_cuda.h -- C ABI of the B200 (sm_100a) Dense-and-Sparse LUT-GEMV hot path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/dsq/kernels.hpp:17-79).  Every entry point
 * below names the reference interface it replaces.  Plain pointers and sizes
 * only; no C++ or torch types cross this boundary; no exception crosses it.
 *
 * Ownership: layer views are non-owning and only read during
 * dsq_cuda_layer_create (pack/re-tile + upload happen once).  The returned
 * layer handle owns all of its device memory.  Caller owns x / y buffers and
 * the stream.  All gemv calls are stream-ordered and asynchronous, and
 * deterministic (no floating-point atomics): a given layer on a given device
 * produces bit-identical outputs on every call.
 *
 * Numerics: LUT centroids, CSR values and activations are fp16 on device
 * (the reference stores fp32 but charges 16 bits: SPEC.md:75, 231).
 * Products are exact (fp16 x fp16 -> fp32), accumulation is fp32.
 */
#ifndef DSQ_CUDA_H
#define DSQ_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSQ_CUDA_ABI_VERSION 1

/* Status codes.  1..15 mirror dsq::errc in declaration order
 * (reference include/dsq/common.hpp:13-29), so a C++ wrapper can rethrow
 * dsq::Error{errc(status-1)} and keep the CLI exit-code mapping of
 * tools/dsq.cpp:399-411 (argument->2, data->3, internal->4). */
typedef enum dsq_status {
    DSQ_OK = 0,
    DSQ_E_MISSING_FILE = 1,
    DSQ_E_MALFORMED_HEADER = 2,
    DSQ_E_NON_FINITE_VALUE = 3,
    DSQ_E_EMPTY_DIMENSION = 4,
    DSQ_E_DIMENSION_OVERFLOW = 5,
    DSQ_E_TRUNCATED_PAYLOAD = 6,
    DSQ_E_CHECKSUM_MISMATCH = 7,
    DSQ_E_UNSUPPORTED_VERSION = 8,
    DSQ_E_SHAPE_MISMATCH = 9,
    DSQ_E_EMPTY_INPUT = 10,
    DSQ_E_INVALID_ARGUMENT = 11,
    DSQ_E_FRACTION_OVERFLOW = 12,
    DSQ_E_EMPTY_CHANNEL = 13,
    DSQ_E_IO_FAILURE = 14,
    DSQ_E_INTERNAL = 15,
    /* device-side failures (no reference counterpart) */
    DSQ_E_CUDA = 100,
    DSQ_E_NO_DEVICE = 101,
    DSQ_E_UNSUPPORTED = 102
} dsq_status;

/* element types for x / y */
typedef enum dsq_dtype { DSQ_F32 = 0, DSQ_F16 = 1, DSQ_F64 = 2 } dsq_dtype;

/* kernel selector, mirrors dsq::BenchKernel (kernels.hpp:71) */
typedef enum dsq_kernel {
    DSQ_KERNEL_LUT = 0,       /* lut_matvec: dense LUT part only        */
    DSQ_KERNEL_CSR = 1,       /* csr_matvec: sparse deltas only          */
    DSQ_KERNEL_FUSED = 2,     /* fused_dns_matvec: LUT + CSR, one launch */
    DSQ_KERNEL_REFERENCE = 3  /* fp16 dense GEMV on the dequantized W    */
} dsq_kernel;

/* Non-owning view of dsq::PackedDense (packfmt.hpp:16-33): the reference
 * layout -- per-row LSB-first index bitstream, row_stride = ceil(cols*bits/8)
 * bytes, LUT rows*groups_per_row*2^bits centroids.  Exactly one of
 * luts_f32 / luts_f16 must be non-null. */
typedef struct dsq_packed_view {
    uint32_t bits;
    uint32_t rows;
    uint32_t cols;
    uint32_t groups_per_row;
    const float* luts_f32;
    const uint16_t* luts_f16; /* IEEE binary16 bit patterns */
    const uint8_t* payload;
    size_t payload_len;       /* must equal rows * row_stride */
} dsq_packed_view;

/* Non-owning view of dsq::CsrMatrix (dns.hpp:14-24).  values are the DELTAS
 * (original - lut_row[0]) written by quantize_layer (pipeline.cpp:25-32).
 * Exactly one of values_f32 / values_f16 must be non-null (may both be null
 * when nnz == 0). */
typedef struct dsq_csr_view {
    uint32_t rows;
    uint32_t cols;
    uint32_t nnz;
    const uint32_t* row_ptr; /* rows + 1 */
    const uint16_t* col_idx; /* nnz, strictly increasing per row */
    const float* values_f32;
    const uint16_t* values_f16;
} dsq_csr_view;

/* Non-owning view of dsq::QuantizedLayer (packfmt.hpp:50-61).  The hybrid
 * split (dns.hpp:55-62) is not passed: it is a deterministic function of
 * `sparse` (container.cpp:138-139) and the device schedule balances outlier
 * skew itself, so fused == fused(top_k=0) == fused(top_k). */
typedef struct dsq_layer_view {
    const char* name;
    uint32_t rows;
    uint32_t cols;
    dsq_packed_view packed;
    dsq_csr_view sparse;
    uint32_t hybrid_top_k; /* recorded for accounting only */
} dsq_layer_view;

typedef struct dsq_cuda_layer dsq_cuda_layer;

/* Layer facts after upload. */
typedef struct dsq_layer_info {
    uint32_t rows, cols, bits, groups_per_row, nnz;
    uint64_t device_bytes;      /* all device allocations of the handle      */
    uint64_t algorithmic_bytes; /* bytes_touched_estimate (kernels.cpp:205)  */
    uint32_t luts_exact_f16;    /* 1 if every centroid was fp16-representable */
    uint32_t values_exact_f16;  /* 1 if every CSR delta was fp16-representable */
    uint32_t workers;           /* warps in the balanced schedule              */
    uint32_t ctas;              /* grid size of the fused launch               */
} dsq_layer_info;

/* ---- library ---------------------------------------------------------- */
int dsq_cuda_abi_version(void);
/* thread-local message for the last non-OK status (never NULL) */
const char* dsq_cuda_last_error(void);
/* The CUDA runtime's pending (non-sticky) error of the calling thread, cleared
 * by the call: 0 when none.  Diagnostics -- every entry point above checks and
 * reports its own CUDA calls. */
int dsq_cuda_pending_error(void);

/* ---- layer lifetime ----------------------------------------------------- */
/* Validates the view exactly like QuantizedLayer::validate()
 * (packfmt.cpp:82-92, dns.cpp:10-29) -- once, here, not per call (the
 * reference validates inside every product, kernels.cpp:52,70,110) --
 * re-tiles the index stream for coalesced per-warp tiles, converts LUTs and
 * deltas to fp16, builds the balanced work schedule and uploads. */
int dsq_cuda_layer_create(const dsq_layer_view* view, int device, dsq_cuda_layer** out);
int dsq_cuda_layer_destroy(dsq_cuda_layer* layer);
int dsq_cuda_layer_get_info(const dsq_cuda_layer* layer, dsq_layer_info* info);

/* ---- products (device buffers, stream-ordered) -------------------------- */
/* y[r] (rows) = product of row r with x (cols).  x_dtype F32/F16 (F32 is
 * rounded to fp16 on device), y_dtype F32/F16.  batch 1..16 (bits 3/4): x
 * [batch][cols] F16 with 16-byte aligned rows, y [batch][rows]; batch 2..4
 * run on the persistent kernel with every decoded weight shared by all
 * vectors, 5..16 on the batched LUT-GEMM K11 plus its finish kernel (two
 * launches; a layer's batched scratch is reused, so one batched product per
 * layer at a time, in stream order).
 * Replaces:
 *   DSQ_KERNEL_LUT   -> dsq::lut_matvec        kernels.hpp:20 / kernels.cpp:51-67
 *   DSQ_KERNEL_CSR   -> dsq::csr_matvec        kernels.hpp:24 / kernels.cpp:69-85
 *   DSQ_KERNEL_FUSED -> dsq::fused_dns_matvec  kernels.hpp:31 / kernels.cpp:108-141
 *   DSQ_KERNEL_REFERENCE -> dense_matvec over ref::dequant_dense (the
 *       "reference" bench kernel, kernels.cpp:227-228,276-278); the dense
 *       fp16 W is materialized on first use. */
int dsq_cuda_gemv(const dsq_cuda_layer* layer, int kernel, const void* x, int x_dtype,
                  void* y, int y_dtype, uint32_t batch, void* stream);
/* convenience wrappers */
int dsq_cuda_lut_gemv(const dsq_cuda_layer* layer, const void* x, int x_dtype, void* y,
                      int y_dtype, uint32_t batch, void* stream);
int dsq_cuda_csr_gemv(const dsq_cuda_layer* layer, const void* x, int x_dtype, void* y,
                      int y_dtype, uint32_t batch, void* stream);
int dsq_cuda_fused_gemv(const dsq_cuda_layer* layer, const void* x, int x_dtype, void* y,
                        int y_dtype, uint32_t batch, void* stream);

/* Plain fp16 dense GEMV (dsq::dense_matvec, kernels.hpp:35 / kernels.cpp:87-106)
 * on a device row-major W[rows][cols]. */
int dsq_cuda_dense_gemv(const uint16_t* w_f16, uint32_t rows, uint32_t cols, const void* x,
                        int x_dtype, void* y, int y_dtype, void* stream);

/* ---- host-buffer products (the reference-facing call) -------------------- */
/* Same semantics as the reference entry points, which take a host
 * std::vector<float> x and return a host std::vector<double> (kernels.hpp:20-32):
 * x_host fp32 [cols] -> y_host fp64 [rows].  Includes the H2D copy of x, the
 * launch and the D2H copy of y; synchronous on the layer's internal stream. */
int dsq_cuda_matvec_host(const dsq_cuda_layer* layer, int kernel, const float* x_host,
                         double* y_host);

/* ---- one-shot host products of the reference's free functions -------------
 * (the C++ drop-ins sqz::lut_matvec / csr_matvec / dense_matvec /
 * dequantize_layer in dsq_cuda.hpp call these; fp32 host x -> fp64 host y)
 *   dsq_cuda_packed_matvec_host -> dsq::lut_matvec(PackedDense, x)  kernels.hpp:20
 *   dsq_cuda_csr_matvec_host    -> dsq::csr_matvec(CsrMatrix, x)    kernels.hpp:24
 *   dsq_cuda_dense_matvec_host  -> dsq::dense_matvec(m, rows, cols, x) kernels.hpp:35
 *     (fp32 weights, fp64 accumulation of the exact fp32 products)
 *   dsq_cuda_dequantize_layer   -> dsq::dequantize_layer(layer)     pipeline.cpp:49-75
 *     w[rows*cols] fp32 = LUT value, and lut_row[0] + delta (one fp32 add)
 *     at every CSR position; bit-equal to the reference for fp16-exact
 *     LUTs/deltas (dsq_layer_info.luts_exact_f16 / values_exact_f16). */
int dsq_cuda_packed_matvec_host(const dsq_packed_view* packed, const float* x_host,
                                double* y_host, int device);
int dsq_cuda_csr_matvec_host(const dsq_csr_view* sparse, const float* x_host, double* y_host,
                             int device);
int dsq_cuda_dense_matvec_host(const float* m_host, uint32_t rows, uint32_t cols,
                               const float* x_host, double* y_host, int device);
int dsq_cuda_dequantize_layer(const dsq_cuda_layer* layer, float* w_dev, void* stream);
int dsq_cuda_dequantize_layer_host(const dsq_cuda_layer* layer, float* w_host);

/* ---- debug / parity kernels ----------------------------------------------- */
/* K5: device decode of the re-tiled index layout into the reference
 * AssignmentVector order (unpack, packfmt.cpp:57-80): assign[rows*cols] u16 */
int dsq_cuda_unpack(const dsq_cuda_layer* layer, uint16_t* assign_dev, void* stream);
/* K6: device dequantization (ref::dequant_dense, kernels.cpp:149-159):
 * w[rows*cols] as fp16 bit patterns (out_dtype F16) or fp32 (F32) */
int dsq_cuda_dequant(const dsq_cuda_layer* layer, void* w_dev, int out_dtype, void* stream);
/* The fp16 A fragments of the hot product kernels (the same PRMT byte-plane
 * decode the stack kernel times, stack.cu dump_frags) scattered back to a
 * dense w[rows*cols] of fp16 bit patterns: equal, bit for bit, to
 * ref::dequant_dense (kernels.cpp:149-159).  3/4-bit layers only
 * (DSQ_E_UNSUPPORTED otherwise). */
int dsq_cuda_dump_frags(const dsq_cuda_layer* layer, uint16_t* w_dev, void* stream);

/* ---- accounting --------------------------------------------------------- */
/* bytes_touched_estimate (kernels.cpp:205-212): the algorithmic bytes of one
 * fused product; group_size 0 = channel-wise (packfmt.cpp:98-121) */
uint64_t dsq_bytes_touched_estimate(uint32_t rows, uint32_t cols, uint32_t bits,
                                    uint32_t group_size, uint64_t nnz);

/* ---- stack runner (decode-time chain of layers) --------------------------- */
/* Runs n layers back to back on one stream with programmatic dependent
 * launch, layer i reading x_i and writing y_i (device pointers, fp16 x,
 * y dtype per y_dtype).  x_i may alias y_{i-1} (chained decode). */
int dsq_cuda_gemv_many(dsq_cuda_layer* const* layers, uint32_t n, int kernel,
                       const void* const* xs, int x_dtype, void* const* ys, int y_dtype,
                       void* stream);

/* ---- persistent stack (K7): a whole decode chain in ONE launch ----------- */
/* Binds n layers (bits 3 or 4, same width, same device) into a dependency
 * chain executed by one persistent kernel: layer i reads x_i -- either the
 * external fp16 vector xs[i] (deps[i] < 0) or the output of layer deps[i]
 * (< i; then y_dtype must be F16) -- and writes ys[i].  Weight streaming runs
 * ahead across layer boundaries; each dependency is a grid-wide completion
 * counter.  Buffers are bound at create time (like a CUDA graph); x/y
 * contents may change between runs.  A layer must not overwrite a buffer
 * that a layer it does not (transitively) depend on still reads.
 * No reference counterpart: the reference runs one product per call
 * (kernels.hpp:31); this is the decode-time caller of that product. */
typedef struct dsq_cuda_stack dsq_cuda_stack;
int dsq_cuda_stack_create(dsq_cuda_layer* const* layers, uint32_t n, const int32_t* deps,
                          const void* const* xs, void* const* ys, int y_dtype,
                          dsq_cuda_stack** out);
/* A stack over `batch` (1..16) activation vectors at once (serving several
 * sequences): vector v of layer i's input is xs[i] + v * x_bstride halves
 * (external inputs) or its producer's output vector v; vector v of the output
 * is ys[i] + v * y_bstride elements (strides multiples of 8, >= the largest
 * cols / rows).  Every decoded weight is shared by all vectors (batch 2: the
 * spare HMMA B columns; 3..4: a second HMMA per fragment).  Batches of 5..16,
 * or of 2..4 whose x vectors do not fit next to the persistent kernel's ring,
 * run in the sequential form: one batched product per layer, back to back
 * under programmatic dependent launch, captured into a CUDA graph during the
 * first run and replayed as one graph launch afterwards (dsq_cuda_stack_info).
 * Single GPU. */
int dsq_cuda_stack_create_batch(dsq_cuda_layer* const* layers, uint32_t n, const int32_t* deps,
                                const void* const* xs, void* const* ys, int y_dtype,
                                uint32_t batch, uint32_t x_bstride, uint32_t y_bstride,
                                dsq_cuda_stack** out);
int dsq_cuda_stack_run(dsq_cuda_stack* stack, void* stream);
/* Serving loop: a stack of K decode steps as ONE resident launch that the
 * host feeds step by step -- no CUDA call, launch or stream synchronisation
 * per step.  gate[i] = k > 0 marks layer i (an external-input layer, deps[i]
 * = -1, its xs[i] = the x_dev given to serve_begin) as reading step k's
 * input (gates non-decreasing); notify[i] = k marks the layer whose
 * completion ends step k (values 1, 2, .. K in layer order, 0 elsewhere).
 *   dsq_cuda_serve_begin: launch (the kernel streams the weights and waits at
 *     the first gate); x_bytes (multiple of 16) per step go to x_dev, and the
 *     first y_bytes of each notify layer's output (16-byte aligned) reach
 *     y_host (any host memory) -- read them after dsq_cuda_serve_step returns;
 *   dsq_cuda_serve_step: copy x_host into a pinned staging buffer and ring
 *     step k's doorbell (host memory); CTA 0 of the kernel copies the bytes
 *     over PCIe into x_dev and releases the grid; the notify layer's
 *     finishing warps write their rows straight into pinned host memory as
 *     64-bit {4 payload bytes, tag k} words (no fence, no gather); returns
 *     once every word of step k carries its tag, the payloads copied into
 *     y_host (with y_bytes = 0: once the kernel's completion word arrives);
 *   dsq_cuda_serve_end: release any steps not fed, wait for the launch.
 * Gated layers of step k must sit after notify k-1 and before notify k
 * (gate[i] == 1 + the notify layers before i) and share one x buffer of
 * their common cols; x_bytes must be cols*2 rounded up to at most 16.  The
 * kernel waits for a step's doorbell without a timeout (an idle server may
 * wait any time; it never computes on a stale x); dsq_cuda_serve_step gives
 * up with DSQ_E_INTERNAL after 10 s without the step's outputs, and
 * dsq_cuda_serve_end releases the steps not fed.  Single GPU, batch 1;
 * dsq_cuda_stack_run is refused on a served stack. */
int dsq_cuda_stack_create_served(dsq_cuda_layer* const* layers, uint32_t n, const int32_t* deps,
                                 const void* const* xs, void* const* ys, int y_dtype,
                                 const uint32_t* gate, const uint32_t* notify,
                                 dsq_cuda_stack** out);
int dsq_cuda_serve_begin(dsq_cuda_stack* stack, void* x_dev, size_t x_bytes, void* y_host,
                         size_t y_bytes, void* stream);
int dsq_cuda_serve_step(dsq_cuda_stack* stack, const void* x_host);
int dsq_cuda_serve_end(dsq_cuda_stack* stack);
/* persistent = 1 when the whole stack runs as one persistent launch, 0 for the
 * sequential form; launches = kernel launches of the last run (1 persistent). */
int dsq_cuda_stack_info(const dsq_cuda_stack* stack, uint32_t* persistent, uint32_t* launches);
/* one decode step from host buffers: copy x_host (x_bytes) into x_dev (the
 * stack's external input), run the stack, copy y_dev into y_host, synchronise
 * the stream.  A 0 byte count skips that copy.  Pinned (device-mapped) x_host
 * with 16-byte aligned buffers and size is read by the GPU itself in a small
 * upload kernel that the stack launch overlaps (programmatic dependent
 * launch); other host memory goes through cudaMemcpyAsync. */
int dsq_cuda_stack_run_host(dsq_cuda_stack* stack, const void* x_host, void* x_dev,
                            size_t x_bytes, const void* y_dev, void* y_host, size_t y_bytes,
                            void* stream);
int dsq_cuda_stack_destroy(dsq_cuda_stack* stack);

/* ---- tensor-parallel sharding (host) ------------------------------
 * dsq_split_range: [lo, hi) of an even split of n into `world` parts on
 *   `align` boundaries (the split every rank computes identically).
 * dsq_shard_rows (column-parallel: q/k/v/gate/up): output rows [lo, hi); the
 *   rows' packed indices, LUTs and CSR rows move with them.
 * dsq_shard_cols (row-parallel: o/down): input columns [lo, hi) (align 32
 *   keeps whole index groups); indices re-packed in the reference LSB-first
 *   layout (packfmt.cpp:40-53), LUTs replicated, CSR filtered and rebased;
 *   channel-wise LUTs only (DSQ_E_UNSUPPORTED otherwise).
 * dsq_shard_decoder: the 7 shards of one decoder layer given in the order
 *   v, q, o, k, up, gate, down (o and down row-parallel, the rest
 *   column-parallel), out[7].
 * A shard owns its arrays; dsq_shard_get returns a view into them (valid
 * until dsq_shard_destroy) that dsq_cuda_layer_create accepts, and lo/hi. */
typedef struct dsq_shard dsq_shard;
int dsq_split_range(uint32_t n, uint32_t world, uint32_t rank, uint32_t align, uint32_t* lo,
                    uint32_t* hi);
int dsq_shard_rows(const dsq_layer_view* layer, uint32_t rank, uint32_t world, uint32_t align,
                   dsq_shard** out);
int dsq_shard_cols(const dsq_layer_view* layer, uint32_t rank, uint32_t world, uint32_t align,
                   dsq_shard** out);
int dsq_shard_decoder(const dsq_layer_view* layers, uint32_t rank, uint32_t world,
                      uint32_t align, dsq_shard** out);
int dsq_shard_get(const dsq_shard* shard, dsq_layer_view* view, uint32_t* lo, uint32_t* hi);
int dsq_shard_destroy(dsq_shard* shard);

/* ---- tensor parallelism: the all-reduce fused into the stack -- */
/* One context per rank (one process per GPU): a receive buffer for the
 * partial outputs of row-parallel layers ([2][world][max_rows] 64-bit words
 * {fp32 value, u32 tag}, single-copy atomic, so no separate flag) and
 * per-CTA arrival flags, shared with the peers through CUDA IPC
 * (ipc_handle_out: 64 bytes, cudaIpcMemHandle_t; exchange them with any
 * out-of-band channel, e.g. torch.distributed all_gather, then
 * dsq_cuda_tp_connect with all world handles in rank order).  No reference
 * counterpart (the reference is single-process). */
typedef struct dsq_cuda_tp dsq_cuda_tp;
int dsq_cuda_tp_create(int device, uint32_t world, uint32_t rank, uint32_t max_rows,
                       uint32_t max_grid, dsq_cuda_tp** out, void* ipc_handle_out);
int dsq_cuda_tp_connect(dsq_cuda_tp* tp, const void* handles);
/* single-process: contexts of one process (same or P2P-capable devices) */
int dsq_cuda_tp_connect_local(dsq_cuda_tp* const* ctxs, uint32_t world);
/* DSQ_OK, or DSQ_E_INTERNAL if a fused reduce gave up waiting for a peer
 * (~4 s watchdog: ranks must run the same launch sequence) */
int dsq_cuda_tp_error(const dsq_cuda_tp* tp);
int dsq_cuda_tp_destroy(dsq_cuda_tp* tp);
/* A stack whose layers with reduce[i] != 0 produce partial sums (row-parallel
 * shards): the finishing CTAs write their partial rows to every rank's
 * receive buffer over NVLink peer memory, signal the same CTA index on every
 * rank (release, system scope), wait for all ranks, and store the sum in rank
 * order as y_i -- no NCCL call and no extra launch on the data path.  All
 * ranks must create the same stacks (same grid) and run them in the same
 * order.  grid = CTAs (0: one per SM). */
int dsq_cuda_stack_create_tp(dsq_cuda_layer* const* layers, uint32_t n, const int32_t* deps,
                             const void* const* xs, void* const* ys, int y_dtype,
                             const uint8_t* reduce, dsq_cuda_tp* tp, uint32_t grid,
                             dsq_cuda_stack** out);

/* ---- quantized-model containers ("DSQCONT1") ----------------------------- */
/* The on-disk input of the hot path: load_container (reference
 * src/container.cpp:181-223, read_layer :102-142) -- magic, version, CRC-32,
 * little-endian fields, per-layer QuantizedLayer::validate -- with the same
 * error codes, then every layer is uploaded (dsq_cuda_layer_create; the fp32
 * centroids / deltas are rounded to fp16, dsq_layer_info reports exactness). */
typedef struct dsq_container_meta {
    uint32_t bits;               /* QuantConfig (container.cpp:150-158)        */
    double sensitive_fraction;
    double outlier_fraction;
    uint32_t group_size;
    uint32_t kmeans_max_iters;
    double kmeans_tol;
    uint64_t seed;
    uint32_t hybrid_top_k;
    uint32_t method_code;
    uint32_t n_layers;
} dsq_container_meta;

typedef struct dsq_cuda_container dsq_cuda_container;
/* parse + validate only (host, no device): the reference's load_container
 * checks, for tools and tests */
int dsq_container_check(const char* path, dsq_container_meta* meta);
int dsq_cuda_container_open(const char* path, int device, dsq_cuda_container** out);
int dsq_cuda_container_meta(const dsq_cuda_container* c, dsq_container_meta* meta);
/* borrowed handles, valid until dsq_cuda_container_close */
dsq_cuda_layer* dsq_cuda_container_layer(const dsq_cuda_container* c, uint32_t index);
const char* dsq_cuda_container_layer_name(const dsq_cuda_container* c, uint32_t index);
int dsq_cuda_container_close(dsq_cuda_container* c);

/* ---- roofline model (reference include/dsq/roofline.hpp:10-88) ----------- */
/* The reference's analytical decode-step model (src/roofline.cpp:10-209,
 * `dsq profile` tools/dsq.cpp:220-271) with the same formulas and errors
 * (invalid_argument for bad shapes / profiles, missing_file and
 * malformed_header from the JSON loaders), a B200 HardwareProfile, and the
 * cost of one fused Dense-and-Sparse LUT-GEMV of the path. */
typedef struct dsq_hw_profile {
    char name[64];
    double peak_flops;     /* operations per second */
    double mem_bandwidth;  /* bytes per second      */
} dsq_hw_profile;

typedef struct dsq_model_shape {
    char name[64];
    uint32_t num_layers, hidden_dim, ffn_dim, num_heads, vocab_size;
    uint32_t seq_len;          /* reference default 128 */
    uint32_t weight_bits;      /* 2..16                 */
    uint32_t activation_bits;  /* fixed 16              */
} dsq_model_shape;

enum { DSQ_LAYER_FC = 0, DSQ_LAYER_ATTENTION = 1, DSQ_LAYER_OTHER = 2 };
/* entries of dsq_decode_step_costs: qkv_proj, out_proj, ffn_gate, ffn_up,
 * ffn_down, lm_head, attn_kv, other */
#define DSQ_DECODE_COSTS 8

typedef struct dsq_layer_cost {
    char name[32];
    int kind;               /* DSQ_LAYER_* */
    double flops, weight_elems, activation_elems, weight_bytes, activation_bytes;
    double predicted_s;     /* max(flops / peak_flops, bytes / mem_bandwidth) */
    int memory_bound;       /* bytes / bw >= flops / peak                     */
    double intensity;       /* flops per memory element (0 if undefined)      */
} dsq_layer_cost;

/* costs[DSQ_DECODE_COSTS]; total / weight_traffic_share may be NULL */
int dsq_decode_step_costs(const dsq_model_shape* shape, const dsq_hw_profile* hw,
                          dsq_layer_cost* costs, dsq_layer_cost* total,
                          double* weight_traffic_share);
int dsq_arithmetic_intensity(const dsq_layer_cost* cost, double* out);
/* predicted decode-step seconds per weight bit width, and normalised to 16-bit */
int dsq_predicted_runtime_curve(const dsq_model_shape* shape, const dsq_hw_profile* hw,
                                const uint32_t* bits, uint32_t n, double* seconds,
                                double* normalized);
int dsq_affine_fit_r2(const uint32_t* bits, const double* normalized, uint32_t n, double* r2);
/* JSON files: {"name", "peak_flops", "mem_bandwidth_bytes_per_s"} and
 * {"name", "num_layers", "hidden_dim", "ffn_dim", "num_heads", "vocab_size",
 *  ["seq_len"], ["weight_bits"]} (roofline.cpp:171-209) */
int dsq_load_hardware_profile(const char* path, dsq_hw_profile* out);
int dsq_load_model_shape(const char* path, dsq_model_shape* out);
/* B200 from MEASURED_PEAKS.json ("hbm_gbs", "bf16_tflops"; NULL or absent:
 * the fallback 6.65 TB/s, 1.59 PFLOP/s) */
int dsq_hw_profile_b200(const char* measured_peaks_json, dsq_hw_profile* out);
/* one fused LUT-GEMV (rows x cols, bits, nnz outliers, batch): charged bytes
 * of kernels.cpp:205-212 (x / y per batch row), 2*B*(rows*cols+nnz) flops */
int dsq_gemv_cost(uint32_t rows, uint32_t cols, uint32_t bits, uint64_t nnz, uint32_t batch,
                  const dsq_hw_profile* hw, dsq_layer_cost* out);

/* ---- GPU channel-wise quantization (the step upstream of the path) ------ */
/* dsq::quantize_channelwise (reference src/nuq.cpp:673-779): one codebook of
 * 2^bits centroids per output row (group_size 0) or per column group, by
 * weighted 1-D k-means (weighted_kmeans_1d nuq.cpp:411-502: weighted-quantile
 * init, Lloyd, exact boundary refinement, merge/split escape), unweighted
 * k-means or round-to-nearest levels; masked positions (already in the
 * sparse part) are excluded and get index 0xFFFF.  Bit-identical codebooks,
 * assignments and objectives to the reference (one CTA per group, exact
 * sequential-order reductions).  Host arrays in and out. */
typedef struct dsq_quant_config {  /* dsq::QuantConfig (nuq.hpp:26-37) */
    uint32_t bits;                 /* 2..8                               */
    double sensitive_fraction;     /* [0, 0.05]                          */
    double outlier_fraction;       /* [0, 0.05]                          */
    uint32_t group_size;           /* 0: channel-wise, else divides cols */
    uint32_t kmeans_max_iters;     /* >= 1                               */
    double kmeans_tol;             /* >= 0                               */
    uint64_t seed;
} dsq_quant_config;
enum { DSQ_CODEBOOK_WEIGHTED_KMEANS = 0, DSQ_CODEBOOK_UNWEIGHTED_KMEANS = 1, DSQ_CODEBOOK_RTN = 2 };
/* w, sens: [rows*cols]; mask: [rows*cols] or NULL; centroids out:
 * [rows * groups_per_row * 2^bits]; assign out: [rows*cols] */
/* dsq::decompose (reference src/dns.cpp:73-145) on the GPU: the mask of the
 * ceil(sensitive_fraction*N) most sensitive weights plus the
 * ceil(outlier_fraction*N) largest magnitudes among the rest (ties: lower
 * row-major index), and their CSR (original values).  row_ptr [rows+1];
 * col_idx / values sized >= nnz (*nnz is set even when the capacity is too
 * small).  Same validation and error codes as the reference. */
int dsq_cuda_decompose(const float* w, const float* sens, uint32_t rows, uint32_t cols,
                       const dsq_quant_config* cfg, int device, uint8_t* mask, uint32_t* row_ptr,
                       uint16_t* col_idx, float* values, uint64_t nnz_cap, uint64_t* nnz,
                       uint32_t* sensitive_count, uint32_t* outlier_count, float* t_min,
                       float* t_max);
int dsq_cuda_quantize_channelwise(const float* w, const float* sens, const uint8_t* mask,
                                  uint32_t rows, uint32_t cols, const dsq_quant_config* cfg,
                                  int method, int device, float* centroids, uint16_t* assign,
                                  double* weighted_objective, double* unweighted_mse_sum);

#ifdef __cplusplus
}
#endif
#endif /* DSQ_CUDA_H */
