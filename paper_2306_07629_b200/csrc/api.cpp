// api.cpp -- the extern "C" boundary (include/dsq_cuda.h): validation,
// re-tiling packer, balanced work scheduler, upload and launches.
//
// Validation mirrors the reference checks and error codes
// (QuantizedLayer::validate packfmt.cpp:82-92, PackedDense::validate
// packfmt.cpp:7-16, CsrMatrix::validate dns.cpp:10-29) but runs once at
// upload instead of inside every product (kernels.cpp:52,70,110).
#include <cuda_runtime.h>

#include "bstream.hpp"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <immintrin.h>

#include "../../include/dsq_cuda.h"
#include "layout.hpp"
#include "stack.hpp"

namespace sqz {
size_t fused_smem_bytes(uint32_t bits);
cudaError_t launch_fused(int mode, const LayerParams& P, const WorkTable& Wt, const uint16_t* x,
                         void* y, bool y_f16, uint32_t ctas, cudaStream_t st, bool pdl);
cudaError_t launch_dense(const uint16_t* w, uint32_t rows, uint32_t cols, const uint16_t* x,
                         void* y, bool y_f16, int num_sms, cudaStream_t st, bool pdl);
cudaError_t launch_decode(int mode, const LayerParams& P, void* out, cudaStream_t st);
cudaError_t launch_f32_to_f16(const float* in, uint16_t* out, uint32_t n, cudaStream_t st,
                              bool pdl);
cudaError_t launch_stack(const StackParams& p, cudaStream_t st, bool pdl);
cudaError_t launch_upload_x(const void* host, void* dev, size_t bytes, cudaStream_t st);
cudaError_t launch_apply_deltas(const uint32_t* row_ptr, const uint32_t* csr, const uint16_t* lut,
                                uint32_t K, uint32_t groups, uint32_t gcols, uint32_t rows,
                                uint32_t cols, float* w, cudaStream_t st);
cudaError_t launch_grouped(int mode, const GroupedParams& p, const uint16_t* x, void* y, bool y_f16,
                           cudaStream_t st, bool pdl);
cudaError_t launch_grouped_decode(int mode, const GroupedParams& p, void* out, cudaStream_t st);
cudaError_t launch_dense_f32(const float* w, uint32_t rows, uint32_t cols, const float* x,
                             double* y, int num_sms, cudaStream_t st);
cudaError_t launch_dump_frags(uint32_t bits, const uint32_t* idx, const uint32_t* lut,
                              uint32_t rows, uint32_t cols, uint32_t tiles, uint32_t ns,
                              uint16_t* out, cudaStream_t st);
cudaError_t launch_decode_tiles(int mode, uint32_t bits, const uint32_t* idx, const uint32_t* lut,
                                uint32_t rows, uint32_t cols, uint32_t ns, void* out,
                                cudaStream_t st);
}  // namespace sqz

using namespace sqz;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(DSQ_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                          \
    do {                                                        \
        cudaError_t _e = (expr);                                \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);     \
    } while (0)

// --- IEEE binary16 <-> binary32 on the host (round to nearest even) --------
uint16_t f32_to_f16(float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u;
    const uint32_t absx = x & 0x7fffffffu;
    if (absx >= 0x7f800000u) return uint16_t(sign | 0x7c00u | (absx > 0x7f800000u ? 0x200u : 0u));
    if (absx >= 0x477ff000u) return uint16_t(sign | 0x7c00u);  // rounds to >= 65520 -> inf
    if (absx < 0x38800000u) {                                   // fp16 subnormal / zero
        if (absx < 0x33000000u) return uint16_t(sign);          // < 2^-25 -> 0
        const uint32_t e = absx >> 23;
        const uint32_t m = (absx & 0x7fffffu) | 0x800000u;
        const uint32_t shift = 126u - e;  // 14..24
        uint32_t h = m >> shift;
        const uint32_t rem = m & ((1u << shift) - 1u);
        const uint32_t half = 1u << (shift - 1);
        if (rem > half || (rem == half && (h & 1u))) ++h;
        return uint16_t(sign | h);
    }
    uint32_t h = ((absx - 0x38000000u) >> 13);
    const uint32_t rem = absx & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
    return uint16_t(sign | h);
}

float f16_to_f32(uint16_t h) {
    const uint32_t sign = uint32_t(h & 0x8000u) << 16;
    uint32_t e = (h >> 10) & 0x1fu, m = h & 0x3ffu, x;
    if (e == 0) {
        if (m == 0) {
            x = sign;
        } else {
            e = 113;
            while (!(m & 0x400u)) {
                m <<= 1;
                --e;
            }
            x = sign | (e << 23) | ((m & 0x3ffu) << 13);
        }
    } else if (e == 31) {
        x = sign | 0x7f800000u | (m << 13);
    } else {
        x = sign | ((e + 112u) << 23) | (m << 13);
    }
    float f;
    std::memcpy(&f, &x, 4);
    return f;
}

size_t row_stride(uint32_t cols, uint32_t bits) { return (size_t(cols) * bits + 7) / 8; }

// index c of a reference-layout row (packfmt.cpp:40-53, LSB-first)
inline uint32_t ref_index(const uint8_t* row, size_t stride, uint32_t c, uint32_t bits) {
    const size_t bp = size_t(c) * bits;
    const size_t byte = bp >> 3;
    uint32_t v = row[byte];
    if (byte + 1 < stride) v |= uint32_t(row[byte + 1]) << 8;
    return (v >> (bp & 7)) & ((1u << bits) - 1u);
}

// pack the 32 indices of one (row, group) into `bits` words (layout.hpp)
inline void encode_unit(const uint8_t* idx, uint32_t bits, uint32_t* w) {
    if (bits == 3) {
        for (int k = 0; k < 3; ++k) {
            uint32_t v = 0;
            for (int n = 0; n < 8; ++n) {
                uint32_t nib = idx[8 * k + n] & 7u;
                nib |= ((idx[24 + n] >> k) & 1u) << 3;
                v |= nib << (4 * n);
            }
            w[k] = v;
        }
    } else if (bits == 4) {
        for (int k = 0; k < 4; ++k) {
            uint32_t v = 0;
            for (int n = 0; n < 8; ++n) v |= uint32_t(idx[8 * k + n] & 15u) << (4 * n);
            w[k] = v;
        }
    } else {
        for (uint32_t k = 0; k < bits; ++k) w[k] = 0;
        for (int j = 0; j < 32; ++j) {
            const uint32_t bp = uint32_t(j) * bits;
            const uint64_t v = uint64_t(idx[j]) << (bp & 31);
            w[bp >> 5] |= uint32_t(v);
            if ((bp & 31) + bits > 32) w[(bp >> 5) + 1] |= uint32_t(v >> 32);
        }
    }
}

int query_num_sms(int device, int* out) {
    int n = 0;
    cudaError_t e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute(SM count)");
    *out = n;
    return DSQ_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// persistent stack plan: shared-memory carve-up and per-layer chunking
// ---------------------------------------------------------------------------
namespace {

struct StackPlanLayer {
    uint32_t rows, cols, tiles, ns, max_nnz_cta;
};

// CTA c of G owns tiles [c*tq + min(c, tr), ...): tq or tq+1 tiles
inline void tile_share(uint32_t tiles, int G, uint32_t c, uint32_t& t0, uint32_t& nt) {
    const uint32_t tq = tiles / uint32_t(G), tr = tiles % uint32_t(G);
    t0 = c * tq + std::min(c, tr);
    nt = tq + (c < tr ? 1u : 0u);
}

uint32_t max_nnz_per_cta(const std::vector<uint32_t>& rp, uint32_t rows, int G) {
    const uint32_t tiles = ceil_div(rows, kTileRows);
    uint32_t m = 0;
    for (int c = 0; c < G; ++c) {
        uint32_t t0, nt;
        tile_share(tiles, G, uint32_t(c), t0, nt);
        const uint32_t r0 = std::min(t0 * kTileRows, rows);
        const uint32_t r1 = std::min((t0 + nt) * kTileRows, rows);
        m = std::max(m, rp[r1] - rp[r0]);
    }
    return m;
}

constexpr uint64_t kSmallLayerUnits = 200;  // (dev per-layer nca) units per CTA for 8 of 16 warps
// 8 consumer warps (four units per iteration, 128 registers) while a CTA's
// mean share of the stack's layers is at most this many units: the LLaMA-7B
// chain (~190) and the 13B stack (~310, +1.5% over 16 warps); 16 warps for
// the 65B stack (~780)
constexpr uint64_t kEightWarpMeanUnits = 500;

// dev (DSQ_STACK_NCA=1): 16-warp stacks whose small layers run on 8 of the
// warps -- measured slower than an 8-warp kernel on the LLaMA-7B chain (2163
// vs 2328 GB/s) and the 13B stack, so the default keeps one count per stack
bool per_layer_nca_enabled() {
    if (const char* e = std::getenv("DSQ_STACK_NCA")) return atoi(e) != 0;
    return false;
}

void fill_desc(StackLayerDesc& d, const StackPlanLayer& l, uint32_t slot_bytes, uint32_t bits,
               int G, uint32_t consumers) {
    static const bool per_layer_nca = per_layer_nca_enabled();
    d.tq = l.tiles / uint32_t(G);
    d.tr = l.tiles % uint32_t(G);
    d.rows = l.rows;
    d.cols = l.cols;
    d.tiles = l.tiles;
    d.ns = l.ns;
    d.cu = slot_bytes / (unit_words(bits) * 4);
    d.dep = kNoDep;
    d.reduce_ord = kNoDep;
    d.nca = consumers;
    d.nca_shift = consumers == 16 ? 4u : consumers == 8 ? 3u : 2u;
    // (dev, DSQ_STACK_NCA=1) a layer that gives a CTA few units runs on the
    // first 8 of 16 consumer warps
    const uint64_t units = uint64_t(ceil_div(l.tiles, G)) * l.ns;
    if (consumers == 16 && units <= kSmallLayerUnits && per_layer_nca) {
        d.nca = 8;
        d.nca_shift = 3;
    }
}

constexpr uint64_t kRingGrowUnits = 250;  // see plan_stack (ring chunk size)

int plan_stack(const StackPlanLayer* Ls, uint32_t n, int G, uint32_t bits, StackParams& sp,
               uint32_t& gseg_cap, uint32_t nbatch = 1, bool x_shared = false) {
    int dev = 0, smax = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // consumer warps: every warp pays a fixed cost per layer (descriptor,
    // chunk and tile bookkeeping, the HMMA drain at tile changes), so stacks
    // whose layers give a CTA few units (LLaMA-7B 4096-row layers: ~111) run
    // better with 8 consumer warps (twice the units each), big layers with 16
    {
        // 16 warps when any layer is large (the small ones then run on 8 of
        // them, fill_desc), 8 when all are small
        bool any_large = false;
        for (uint32_t i = 0; i < n; ++i)
            any_large |= uint64_t(ceil_div(Ls[i].tiles, G)) * Ls[i].ns > kSmallLayerUnits;
        sp.consumers = any_large && per_layer_nca_enabled() ? kStackConsumersDefault : 8u;
        if (!per_layer_nca_enabled()) {  // the round-1 rule: mean units per layer
            uint64_t units = 0;
            for (uint32_t i = 0; i < n; ++i) units += uint64_t(ceil_div(Ls[i].tiles, G)) * Ls[i].ns;
            sp.consumers = units <= kEightWarpMeanUnits * n ? 8u : kStackConsumersDefault;
        }
    }
    if (const char* e = std::getenv("DSQ_STACK_CONSUMERS")) {
        const int c = atoi(e);
        if (c == 8 || c == 16) sp.consumers = uint32_t(c);
    }
    if (nbatch == 8) sp.consumers = 8;  // four accumulator pairs: 8-consumer kernels only
    uint32_t max_ns = 0, max_rows = 0, max_nnz = 0;
    for (uint32_t i = 0; i < n; ++i) {
        max_ns = std::max(max_ns, Ls[i].ns);
        max_rows = std::max(max_rows, ceil_div(Ls[i].tiles, G) * kTileRows);
        max_nnz = std::max(max_nnz, Ls[i].max_nnz_cta);
    }
    // CSR warps: 2 while a CTA's CSR work (entries x batch vectors, each
    // vector is one scan) stays small -- the 0.05-0.45% outlier loads at
    // batch 1 -- else 4 (DSQ_STACK_CSR_WARPS: dev override)
    sp.csr_warps = uint64_t(max_nnz) * nbatch <= 1536 ? 2u : 4u;
    if (const char* e = std::getenv("DSQ_STACK_CSR_WARPS")) {
        const int c = atoi(e);
        if (c >= 1 && c <= 4) sp.csr_warps = uint32_t(c);
    }
    auto al = [](size_t b, size_t a) { return (b + a - 1) / a * a; };
    // per-layer buffers: two (layer l uses buffer l & 1, so loading layer
    // l+1 overlaps layer l), one for a single-layer plan (more ring)
    const size_t nbuf = n == 1 ? 1 : 2;
    sp.nbuf = uint32_t(nbuf);
    size_t off = 1024;  // mbarriers
    sp.off_desc = uint32_t(off);
    off += 8 * 128;     // descriptor cache (stack.cu)
    sp.off_x = uint32_t(off);
    sp.nbatch = nbatch;
    sp.nvec = nbatch;
    sp.xvec = uint32_t(size_t(max_ns) * kSpanCols);  // halves per vector, largest layer
    sp.x_bytes = uint32_t(size_t(sp.xvec) * 2 * nbatch);
    // x: layer l takes ns_l * 256 halves per vector; two consecutive layers
    // must coexist (layer l+1's x is staged while layer l decodes): a region
    // of the largest consecutive pair, even layers at its bottom, odd at its
    // top (stack.cu x_region) -- not two buffers of the largest layer
    size_t x_pair = 0;
    for (uint32_t i = 1; i < n; ++i)
        x_pair = std::max(x_pair, (size_t(Ls[i - 1].ns) + Ls[i].ns) * kSpanCols * 2 * nbatch);
    const bool two = nbuf == 2 && !x_shared;
    sp.x_step = two ? uint32_t(x_pair) : 0u;
    off += two ? x_pair : size_t(sp.x_bytes);
    sp.off_lut = uint32_t(off);
    sp.lut_bytes = uint32_t(al(size_t(max_rows) * tile_lut_words(bits) * 4, 128));
    off += nbuf * size_t(sp.lut_bytes);
    sp.off_rp = uint32_t(off);
    sp.rp_words = uint32_t(al(max_rows + 1, 32));
    off += nbuf * size_t(sp.rp_words) * 4;
    sp.off_csr = uint32_t(off);
    sp.csr_cap = uint32_t(al(std::min<uint32_t>(std::max<uint32_t>(max_nnz + 4, 32), 2048), 32));
    off += nbuf * size_t(sp.csr_cap) * 4;
    sp.off_hb = uint32_t(off);
    sp.hb_words = (sp.csr_cap / 32 + 16 + 3) & ~3u;  // 16-byte aligned TMA destinations
    off += nbuf * size_t(sp.hb_words) * 4;
    sp.off_part = uint32_t(off);
    sp.part_rows = std::max<uint32_t>(max_rows, kTileRows);
    off = al(off + nbuf * size_t(nbatch) * sp.part_rows * sp.consumers * 4, 128);
    sp.off_seg = uint32_t(off);
    sp.seg_cap = sp.csr_cap + 128;  // one float per staged entry position (+ a round)
    off += nbuf * size_t(nbatch) * sp.seg_cap * 4;
    gseg_cap = max_nnz > sp.csr_cap - 4 ? uint32_t(al(max_nnz + 256, 4)) : 0;
    sp.off_ring = uint32_t(al(off, 1024));
    // the rest is the consumers' private rings: 2 slots per consumer warp,
    // each a whole number of units (384 B 3-bit, 512 B 4-bit)
    const uint32_t ub = unit_words(bits) * 4;
    const size_t ring = size_t(smax) > sp.off_ring ? size_t(smax) - sp.off_ring : 0;
    uint32_t ws = kWarpSlotsDefault;
    if (const char* e = std::getenv("DSQ_STACK_SLOTS"))
        ws = std::max<uint32_t>(2, std::min<uint32_t>(kMaxWarpSlots, uint32_t(atoi(e))));
    sp.n_slots = sp.consumers * ws;
    sp.slot_bytes = uint32_t(ring / sp.n_slots / ub * ub);
    if (two) {
        // small layers (mean units per CTA < kRingGrowUnits, the LLaMA-7B
        // chain) keep the chunk size of two full-size x buffers: measured
        // -1% on the 7B chain with the larger chunks the pair-sized region
        // frees, +4% on the 13B / 65B stacks (larger layers)
        uint64_t units = 0;
        for (uint32_t i = 0; i < n; ++i) units += uint64_t(ceil_div(Ls[i].tiles, G)) * Ls[i].ns;
        const size_t freed = 2 * size_t(sp.x_bytes) - x_pair;
        if (units < kRingGrowUnits * n && ring > freed) {
            const uint32_t old_slot = uint32_t((ring - freed) / sp.n_slots / ub * ub);
            if (old_slot >= 2 * ub) sp.slot_bytes = old_slot;
        }
    }
    if (sp.slot_bytes < 2 * ub) {
        // large batched x: retry with one shared x buffer before giving up
        if (nbatch > 1 && nbuf == 2 && !x_shared)
            return plan_stack(Ls, n, G, bits, sp, gseg_cap, nbatch, true);
        return fail(DSQ_E_UNSUPPORTED, "stack: layer too large for the shared-memory ring "
                    "(x %u B)", sp.x_bytes);
    }
    sp.smem_bytes = sp.off_ring + sp.n_slots * sp.slot_bytes;
    sp.grid = uint32_t(G);
    sp.bits = bits;
    sp.k29 = 1u << 29;
    sp.k30 = 1u << 30;
    sp.k31 = 1u << 31;
    sp.kneg = 0xffffffffu;
    for (uint32_t i = 0; i < n && i < kInlineLayers; ++i)
        fill_desc(sp.inl[i], Ls[i], sp.slot_bytes, bits, G, sp.consumers);
    return DSQ_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// layer handle
// ---------------------------------------------------------------------------
struct dsq_cuda_layer {
    int device = 0;
    int num_sms = 0;
    std::string name;
    uint32_t rows = 0, cols = 0, bits = 0, groups = 1, nnz = 0, hybrid_top_k = 0;
    uint32_t n_rb = 0, ng = 0, n_workers = 0, ctas = 0;
    uint32_t luts_exact = 1, values_exact = 1;
    uint64_t algorithmic_bytes = 0;
    void* arena = nullptr;      // one device allocation for everything below
    size_t arena_bytes = 0;
    LayerParams P{};
    WorkTable W{};
    uint16_t* x16 = nullptr;    // fp16 staging of an fp32 x
    float* y32 = nullptr;       // host-API output staging
    float* x32 = nullptr;       // host-API input staging
    float* x32_pin = nullptr;   // host-API pinned, device-mapped staging (lazy)
    uint16_t* x16_pin = nullptr;  // host-API: fp16 x converted on the host (F16C)
    uint16_t* x16_map = nullptr;
    cudaGraphExec_t host_graph[4] = {nullptr, nullptr, nullptr, nullptr};  // per kernel
    float* y32_pin = nullptr;
    float* x32_map = nullptr;   // their device addresses
    float* y32_map = nullptr;
    uint16_t* dense_w = nullptr;  // lazily materialized fp16 dense W (reference kernel)
    // tile-record layout (bits 3/4): the persistent stack kernel's format
    bool rec_layout = false;
    bool grouped = false;                   // groups_per_row > 1: reference layout, grouped_gemv
    GroupedParams G{};
    uint32_t tiles = 0, ns = 0;
    const uint32_t* tlut = nullptr;         // LUT planes [tiles][4][LW]
    const uint32_t* rec = nullptr;
    const uint32_t* zero_rp = nullptr;      // all-zero row_ptr (LUT-only products)
    const uint32_t* csr_rng = nullptr;      // [num_sms][2] per-CTA CSR entry ranges
    const uint32_t* zero_rng = nullptr;     // all-zero ranges (LUT-only products)
    const uint32_t* csr_heads = nullptr;    // row-start bitmap of the CSR entries
    std::vector<uint32_t> row_ptr_host;
    StackParams sp1{};                      // single-layer stack plan
    uint32_t* stack_counters = nullptr;     // [2]
    float* gseg1 = nullptr;
    StackParams sp2{}, sp4{}, sp8{};        // batch 2 / 3..4 / 5..8 single-layer plans (lazy)
    bool sp2_ready = false, sp4_ready = false, sp8_ready = false;
    bool sp2_failed = false, sp4_failed = false, sp8_failed = false;  // x does not fit: K11
    bool k7_batch_failed(uint32_t nb) const {
        return nb == 2 ? sp2_failed : nb == 4 ? sp4_failed : sp8_failed;
    }
    float* gseg2 = nullptr;
    float* gseg4 = nullptr;
    float* gseg8 = nullptr;
    cudaStream_t stream = nullptr;
    BStreamDevPlan bs[2] = {};              // K9 plans for B <= 8 / <= 16 (lazy)
    void* bs_mem[2] = {nullptr, nullptr};   // their device allocations
    std::mutex mu;       // guards dense_w materialization and the batched plans
    std::mutex host_mu;  // serializes the host-buffer API on the internal stream
};

// shared with container.cpp (C linkage, not in the public header)
extern "C" int dsq_internal_fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
extern "C" {

int dsq_cuda_abi_version(void) { return DSQ_CUDA_ABI_VERSION; }

const char* dsq_cuda_last_error(void) { return g_err.c_str(); }
int dsq_cuda_pending_error(void) { return int(cudaGetLastError()); }

uint64_t dsq_bytes_touched_estimate(uint32_t rows, uint32_t cols, uint32_t bits,
                                    uint32_t group_size, uint64_t nnz) {
    // packfmt.cpp:98-121 + kernels.cpp:205-212
    const uint64_t weights = uint64_t(rows) * cols;
    uint64_t total_bits;
    if (bits == 16) {
        total_bits = weights * 16;
    } else {
        const uint64_t gpr = group_size == 0 ? 1 : cols / group_size;
        total_bits = uint64_t(rows) * ((uint64_t(cols) * bits + 7) / 8) * 8;
        total_bits += uint64_t(rows) * gpr * (1u << bits) * 16;
        if (nnz > 0) total_bits += nnz * 32 + (uint64_t(rows) + 1) * 32;
    }
    return total_bits / 8 + uint64_t(cols) * 2 + uint64_t(rows) * 2;
}

static int validate_view(const dsq_layer_view* v) {
    if (!v) return fail(DSQ_E_INVALID_ARGUMENT, "null layer view");
    if (!v->name || !v->name[0]) return fail(DSQ_E_INVALID_ARGUMENT, "layer: empty name");
    const dsq_packed_view& p = v->packed;
    // PackedDense::validate (packfmt.cpp:7-16)
    if (p.bits < 1 || p.bits > 8)
        return fail(DSQ_E_INVALID_ARGUMENT, "packed: bits must be in 1..8");
    if (p.rows < 1 || p.cols < 1) return fail(DSQ_E_EMPTY_DIMENSION, "packed: empty dims");
    if (p.groups_per_row < 1 || p.cols % p.groups_per_row != 0)
        return fail(DSQ_E_SHAPE_MISMATCH, "packed: groups_per_row must divide cols");
    if (!p.luts_f32 == !p.luts_f16)
        return fail(DSQ_E_SHAPE_MISMATCH, "packed: exactly one of luts_f32/luts_f16 required");
    if (!p.payload || p.payload_len != size_t(p.rows) * row_stride(p.cols, p.bits))
        return fail(DSQ_E_SHAPE_MISMATCH, "packed: payload size mismatch");
    // CsrMatrix::validate (dns.cpp:10-29)
    const dsq_csr_view& s = v->sparse;
    if (s.cols >= 65536u) return fail(DSQ_E_DIMENSION_OVERFLOW, "csr: cols must be < 65536");
    if (!s.row_ptr) return fail(DSQ_E_SHAPE_MISMATCH, "csr: bad row_ptr length");
    if (s.row_ptr[0] != 0) return fail(DSQ_E_INTERNAL, "csr: row_ptr[0] != 0");
    for (uint32_t r = 0; r < s.rows; ++r) {
        if (s.row_ptr[r] > s.row_ptr[r + 1])
            return fail(DSQ_E_INTERNAL, "csr: row_ptr not nondecreasing");
        for (uint32_t q = s.row_ptr[r]; q < s.row_ptr[r + 1]; ++q) {
            if (q >= s.nnz) return fail(DSQ_E_SHAPE_MISMATCH, "csr: nnz mismatch");
            if (s.col_idx[q] >= s.cols)
                return fail(DSQ_E_INTERNAL, "csr: column index out of range");
            if (q > s.row_ptr[r] && s.col_idx[q - 1] >= s.col_idx[q])
                return fail(DSQ_E_INTERNAL, "csr: columns not strictly increasing");
        }
    }
    if (s.row_ptr[s.rows] != s.nnz) return fail(DSQ_E_SHAPE_MISMATCH, "csr: nnz mismatch");
    if (s.nnz > 0 && (!s.col_idx || (!s.values_f32 == !s.values_f16)))
        return fail(DSQ_E_SHAPE_MISMATCH, "csr: exactly one of values_f32/values_f16 required");
    for (uint32_t q = 0; q < s.nnz; ++q) {
        const float f = s.values_f32 ? s.values_f32[q] : f16_to_f32(s.values_f16[q]);
        if (!std::isfinite(f)) return fail(DSQ_E_NON_FINITE_VALUE, "csr: non-finite value");
    }
    // QuantizedLayer::validate (packfmt.cpp:82-92)
    if (p.rows != v->rows || p.cols != v->cols)
        return fail(DSQ_E_SHAPE_MISMATCH, "%s: packed dims mismatch", v->name);
    if (s.rows != v->rows || s.cols != v->cols)
        return fail(DSQ_E_SHAPE_MISMATCH, "%s: sparse dims mismatch", v->name);
    return DSQ_OK;
}

int dsq_internal_validate_view(const dsq_layer_view* v) { return validate_view(v); }

// Grouped-LUT layers (groups_per_row > 1, the grouping ablation): the
// reference payload uploaded as is, fp16 LUTs [rows][groups][K], the CSR as
// the other layouts; products by grouped_gemv (kernels.cu), no stack support.
static int create_grouped(const dsq_layer_view* v, int device, int num_sms, dsq_cuda_layer** out) {
    auto* L = new dsq_cuda_layer;
    L->device = device;
    L->num_sms = num_sms;
    L->name = v->name;
    L->rows = v->rows;
    L->cols = v->cols;
    L->bits = v->packed.bits;
    L->groups = v->packed.groups_per_row;
    L->nnz = v->sparse.nnz;
    L->hybrid_top_k = v->hybrid_top_k;
    L->grouped = true;
    const uint32_t rows = L->rows, cols = L->cols, bits = L->bits, groups = L->groups;
    const uint32_t K = 1u << bits;
    L->algorithmic_bytes = dsq_bytes_touched_estimate(rows, cols, bits, cols / groups, L->nnz);
    const size_t nl = size_t(rows) * groups * K;
    std::vector<uint16_t> lut(nl);
    for (size_t i = 0; i < nl; ++i) {
        if (v->packed.luts_f16) {
            lut[i] = v->packed.luts_f16[i];
        } else {
            const float f = v->packed.luts_f32[i];
            lut[i] = f32_to_f16(f);
            if (f16_to_f32(lut[i]) != f) L->luts_exact = 0;
        }
        if ((lut[i] & 0x7c00u) == 0x7c00u) {
            delete L;
            return fail(DSQ_E_NON_FINITE_VALUE, "%s: LUT centroid %zu is not finite in fp16",
                        v->name, i);
        }
    }
    std::vector<uint32_t> csr(std::max<uint32_t>(L->nnz, 1), 0);
    for (uint32_t q = 0; q < L->nnz; ++q) {
        uint16_t h;
        if (v->sparse.values_f16) {
            h = v->sparse.values_f16[q];
        } else {
            h = f32_to_f16(v->sparse.values_f32[q]);
            if (f16_to_f32(h) != v->sparse.values_f32[q]) L->values_exact = 0;
        }
        csr[q] = uint32_t(v->sparse.col_idx[q]) | (uint32_t(h) << 16);
    }
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t pay = v->packed.payload_len;
    const size_t o_pay = 0, o_lut = al(pay + 16), o_rp = o_lut + al(nl * 2),
                 o_csr = o_rp + al((size_t(rows) + 1) * 4), o_x16 = o_csr + al(csr.size() * 4),
                 total = o_x16 + al((size_t(cols) + 8) * 2);
    cudaError_t e = cudaMalloc(&L->arena, total);
    if (e != cudaSuccess) {
        delete L;
        return cuda_fail(e, "cudaMalloc(grouped layer)");
    }
    L->arena_bytes = total;
    uint8_t* base = static_cast<uint8_t*>(L->arena);
    if ((e = cudaMemcpy(base + o_pay, v->packed.payload, pay, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(base + o_lut, lut.data(), nl * 2, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(base + o_rp, v->sparse.row_ptr, (size_t(rows) + 1) * 4,
                        cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(base + o_csr, csr.data(), csr.size() * 4, cudaMemcpyHostToDevice)) !=
            cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking)) != cudaSuccess) {
        dsq_cuda_layer_destroy(L);
        return cuda_fail(e, "grouped layer upload");
    }
    L->G = GroupedParams{base + o_pay, reinterpret_cast<const uint16_t*>(base + o_lut),
                         reinterpret_cast<const uint32_t*>(base + o_rp),
                         reinterpret_cast<const uint32_t*>(base + o_csr), rows, cols, bits, groups,
                         cols / groups, uint32_t(row_stride(cols, bits))};
    L->P.row_ptr = L->G.row_ptr;
    L->P.csr = L->G.csr;
    L->P.lut = L->G.lut;
    L->P.rows = rows;
    L->P.cols = cols;
    L->P.bits = bits;
    L->P.nnz = L->nnz;
    L->x16 = reinterpret_cast<uint16_t*>(base + o_x16);
    *out = L;
    return DSQ_OK;
}

int dsq_cuda_layer_create(const dsq_layer_view* v, int device, dsq_cuda_layer** out) {
    if (!out) return fail(DSQ_E_INVALID_ARGUMENT, "null output handle");
    *out = nullptr;
    int rc = validate_view(v);
    if (rc) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(DSQ_E_NO_DEVICE, "no CUDA device visible");
    if (device < 0 || device >= ndev) return fail(DSQ_E_NO_DEVICE, "bad device %d", device);
    CUDA_TRY(cudaSetDevice(device));
    int num_sms = 0;
    if ((rc = query_num_sms(device, &num_sms))) return rc;

    if (v->packed.groups_per_row > 1) return create_grouped(v, device, num_sms, out);
    auto* L = new dsq_cuda_layer;
    L->device = device;
    L->num_sms = num_sms;
    L->name = v->name;
    L->rows = v->rows;
    L->cols = v->cols;
    L->bits = v->packed.bits;
    L->nnz = v->sparse.nnz;
    L->hybrid_top_k = v->hybrid_top_k;
    const uint32_t bits = L->bits, rows = L->rows, cols = L->cols;
    const uint32_t n_rb = ceil_div(rows, kRowBlock), ng = ceil_div(cols, kGroupCols);
    const uint32_t K = 1u << bits;
    L->n_rb = n_rb;
    L->ng = ng;
    L->algorithmic_bytes = dsq_bytes_touched_estimate(rows, cols, bits, 0, L->nnz);

    // ---- LUT -> fp16 [n_rb*32][K]
    std::vector<uint16_t> lut(size_t(n_rb) * kRowBlock * K, 0);
    for (size_t i = 0; i < size_t(rows) * K; ++i) {
        if (v->packed.luts_f16) {
            lut[i] = v->packed.luts_f16[i];
        } else {
            const float f = v->packed.luts_f32[i];
            lut[i] = f32_to_f16(f);
            if (f16_to_f32(lut[i]) != f) L->luts_exact = 0;
        }
        const uint16_t h = lut[i];
        if ((h & 0x7c00u) == 0x7c00u) {
            delete L;
            return fail(DSQ_E_NON_FINITE_VALUE,
                        "%s: LUT centroid %zu is not finite in fp16", v->name, i);
        }
    }
    const size_t stride = row_stride(cols, bits);
    const bool rec_layout = (bits == 3 || bits == 4);
    const uint32_t ntiles = ceil_div(rows, kTileRows), ns = ceil_div(cols, kSpanCols);
    const uint32_t lw = rec_layout ? tile_lut_words(bits) : 0;
    const size_t unit_words_g = size_t(bits) * 32;
    const size_t n_units = size_t(n_rb) * ng;
    std::vector<uint32_t> words, tluts;
    if (rec_layout) {
        // ---- tile layout: LUT planes [tiles][4][lw] + index units [tiles][ns][32 x bits] (stack.hpp)
        words.assign(size_t(ntiles) * ns * unit_words(bits), 0);
        tluts.assign(size_t(ntiles) * kTileRows * lw, 0);
#pragma omp parallel for schedule(dynamic, 4)
        for (int64_t tile = 0; tile < int64_t(ntiles); ++tile) {
            uint8_t idx[32];
            uint32_t w[8];
            for (uint32_t i = 0; i < kTileRows; ++i) {
                const uint32_t r = uint32_t(tile) * kTileRows + i;
                if (r >= rows) break;  // padded rows: zero LUT, index 0
                const uint16_t* e = lut.data() + size_t(r) * K;
                uint32_t* pl = tluts.data() + (size_t(tile) * kTileRows + i) * lw;
                for (uint32_t set = 0; set < K / 8; ++set) {  // planes of entries 8*set .. 8*set+7
                    uint32_t l0 = 0, l1 = 0, h0 = 0, h1 = 0;
                    for (int q = 0; q < 4; ++q) {
                        l0 |= uint32_t(e[8 * set + q] & 0xffu) << (8 * q);
                        l1 |= uint32_t(e[8 * set + 4 + q] & 0xffu) << (8 * q);
                        h0 |= uint32_t(e[8 * set + q] >> 8) << (8 * q);
                        h1 |= uint32_t(e[8 * set + 4 + q] >> 8) << (8 * q);
                    }
                    pl[4 * set + 0] = l0;
                    pl[4 * set + 1] = l1;
                    pl[4 * set + 2] = h0;
                    pl[4 * set + 3] = h1;
                }
                const uint8_t* row = v->packed.payload + size_t(r) * stride;
                for (uint32_t g = 0; g < ns * (kSpanCols / 32); ++g) {
                    const uint32_t s = g / 8, gs = g % 8, h = gs >> 2, t = gs & 3;
                    for (uint32_t j = 0; j < 32; ++j) {
                        const uint32_t c = s * kSpanCols + tile_col(h, t, j);
                        idx[j] = c < cols ? uint8_t(ref_index(row, stride, c, bits)) : 0;
                    }
                    encode_unit(idx, bits, w);
                    const uint32_t lane = 16 * h + 4 * i + t;
                    uint32_t* sp = words.data() + (size_t(tile) * ns + s) * unit_words(bits);
                    for (uint32_t k = 0; k < bits; ++k) {
                        if (bits == 3)
                            sp[k * 32 + lane] = w[k];
                        else
                            sp[lane * 4 + k] = w[k];
                    }
                }
            }
        }
    } else {
        // ---- tiled index words (generic widths, stream-K kernel)
        words.assign(n_units * unit_words_g, 0);
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t rb = 0; rb < int64_t(n_rb); ++rb) {
            uint8_t idx[32];
            uint32_t w[8];
            for (uint32_t lane = 0; lane < kRowBlock; ++lane) {
                const uint32_t r = uint32_t(rb) * kRowBlock + lane;
                const uint8_t* row = r < rows ? v->packed.payload + size_t(r) * stride : nullptr;
                for (uint32_t g = 0; g < ng; ++g) {
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t c = g * kGroupCols + j;
                        idx[j] = (row && c < cols) ? uint8_t(ref_index(row, stride, c, bits)) : 0;
                    }
                    encode_unit(idx, bits, w);
                    uint32_t* dst = words.data() + (size_t(rb) * ng + g) * unit_words_g;
                    for (uint32_t k = 0; k < bits; ++k) dst[k * 32 + lane] = w[k];
                }
            }
        }
    }
    L->rec_layout = rec_layout;
    L->tiles = ntiles;
    L->ns = ns;
    L->row_ptr_host.assign(v->sparse.row_ptr, v->sparse.row_ptr + rows + 1);
    // ---- CSR entries: col | fp16(delta) << 16
    std::vector<uint32_t> csr(std::max<uint32_t>(L->nnz, 1), 0);
    for (uint32_t q = 0; q < L->nnz; ++q) {
        uint16_t h;
        if (v->sparse.values_f16) {
            h = v->sparse.values_f16[q];
        } else {
            const float f = v->sparse.values_f32[q];
            h = f32_to_f16(f);
            if (f16_to_f32(h) != f) L->values_exact = 0;
        }
        if ((h & 0x7c00u) == 0x7c00u) {
            delete L;
            return fail(DSQ_E_NON_FINITE_VALUE, "%s: CSR delta %u is not finite in fp16",
                        v->name, q);
        }
        csr[q] = uint32_t(v->sparse.col_idx[q]) | (uint32_t(h) << 16);
    }
    // ---- balanced schedule (stream-K over units, CSR cost weighted by nnz)
    const double beta = 1.0 / 64.0;  // one CSR entry ~ 1/64 of a 32x32 dense unit
    std::vector<double> rb_cost(n_rb);
    for (uint32_t rb = 0; rb < n_rb; ++rb) {
        const uint32_t r0 = std::min(rb * kRowBlock, rows), r1 = std::min(r0 + kRowBlock, rows);
        const double nz = double(v->sparse.row_ptr[r1] - v->sparse.row_ptr[r0]);
        rb_cost[rb] = 1.0 + beta * nz / ng;  // per unit of this row block
    }
    double total = 0;
    for (uint32_t rb = 0; rb < n_rb; ++rb) total += rb_cost[rb] * ng;
    int ctas_per_sm = kCtasPerSmDefault;
    if (const char* e = std::getenv("DSQ_CTAS_PER_SM")) ctas_per_sm = std::max(1, std::min(3, atoi(e)));
    const uint32_t max_workers =
        std::min<uint32_t>(uint32_t(num_sms) * ctas_per_sm * kWarpsPerCta, kMaxWorkers);
    uint32_t nw = uint32_t(std::max<size_t>(1, std::min<size_t>(max_workers, (n_units + 1) / 2)));
    std::vector<uint32_t> bounds;  // unit boundaries, nw+1 entries
    bounds.reserve(nw + 1);
    {
        bounds.push_back(0);
        double acc = 0;
        uint32_t w = 1;
        for (size_t u = 0; u < n_units && w < nw; ++u) {
            acc += rb_cost[u / ng];
            while (w < nw && acc >= total * double(w) / nw - 1e-9) {
                bounds.push_back(uint32_t(u + 1));
                ++w;
            }
        }
        while (bounds.size() < size_t(nw) + 1) bounds.push_back(uint32_t(n_units));
        bounds.back() = uint32_t(n_units);
    }
    // drop empty ranges -> strictly increasing u0[]
    {
        uint32_t n = 0;
        L->W.u0[0] = 0;
        for (uint32_t w = 0; w < nw; ++w)
            if (bounds[w + 1] > bounds[w]) L->W.u0[++n] = bounds[w + 1];
        nw = n;
        L->W.n = nw;
    }
    {
        L->n_workers = nw;
        L->ctas = ceil_div(nw, kWarpsPerCta);
        const size_t scratch_floats = size_t(2) * nw * kRowBlock;
        // ---- one arena
        auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t o_words = 0;
        const size_t o_tlut = o_words + al(words.size() * 4);
        const size_t o_lut = o_tlut + al(tluts.size() * 4 + 16);
        const size_t o_rowptr = o_lut + al(lut.size() * 2);
        // row_ptr / CSR padded by 16 B: the stack loader copies 16-byte granules
        const size_t o_csr = o_rowptr + al((size_t(rows) + 1) * 4 + 16);
        const size_t o_scratch = o_csr + al(csr.size() * 4 + 16);
        const size_t o_counters = o_scratch + al(scratch_floats * 4);
        const size_t o_x16 = o_counters + al(size_t(n_rb) * 4);
        const size_t o_x32 = o_x16 + al((size_t(ng) * kGroupCols + 8) * 2);
        const size_t o_y32 = o_x32 + al(size_t(cols) * 4);
        const size_t o_zrp = o_y32 + al(size_t(rows) * 4);
        const size_t o_scnt = o_zrp + al((size_t(rows) + 1) * 4 + 16);
        const size_t heads_words = size_t(L->nnz) / 32 + 8;  // row-start bitmap (+pad)
        const size_t o_heads = o_scnt + al(2 * 4);
        const size_t o_rng = o_heads + al(heads_words * 4);   // per-CTA CSR entry ranges
        const size_t o_zrng = o_rng + al(size_t(num_sms) * 8);  // all-zero ranges (LUT-only)
        // single-layer stack plan (bits 3/4)
        uint32_t gseg_cap = 0;
        if (rec_layout) {
            StackPlanLayer pl{rows, cols, ntiles, ns, max_nnz_per_cta(L->row_ptr_host, rows, num_sms)};
            int prc = plan_stack(&pl, 1, num_sms, bits, L->sp1, gseg_cap);
            if (prc) {
                delete L;
                return prc;
            }
        }
        const size_t o_gseg = o_zrng + al(size_t(num_sms) * 8);
        const size_t total_bytes = o_gseg + al(size_t(num_sms) * 2 * gseg_cap * 4 + 4);
        cudaError_t e = cudaMalloc(&L->arena, total_bytes);
        if (e != cudaSuccess) {
            delete L;
            return cuda_fail(e, "cudaMalloc(layer arena)");
        }
        L->arena_bytes = total_bytes;
        uint8_t* base = static_cast<uint8_t*>(L->arena);
        LayerParams& P = L->P;
        P.words = reinterpret_cast<const uint32_t*>(base + o_words);
        P.lut = reinterpret_cast<const uint16_t*>(base + o_lut);
        P.row_ptr = reinterpret_cast<const uint32_t*>(base + o_rowptr);
        P.csr = reinterpret_cast<const uint32_t*>(base + o_csr);
        P.scratch = reinterpret_cast<float*>(base + o_scratch);
        P.counters = reinterpret_cast<uint32_t*>(base + o_counters);
        P.rows = rows;
        P.cols = cols;
        P.bits = bits;
        P.n_rb = n_rb;
        P.ng = ng;
        P.n_workers = nw;
        P.nnz = L->nnz;
        L->x16 = reinterpret_cast<uint16_t*>(base + o_x16);
        L->x32 = reinterpret_cast<float*>(base + o_x32);
        L->y32 = reinterpret_cast<float*>(base + o_y32);
        L->zero_rp = reinterpret_cast<const uint32_t*>(base + o_zrp);
        L->stack_counters = reinterpret_cast<uint32_t*>(base + o_scnt);
        L->gseg1 = reinterpret_cast<float*>(base + o_gseg);
        L->csr_rng = reinterpret_cast<const uint32_t*>(base + o_rng);
        L->zero_rng = reinterpret_cast<const uint32_t*>(base + o_zrng);
        L->csr_heads = reinterpret_cast<const uint32_t*>(base + o_heads);
        std::vector<uint32_t> heads(heads_words, 0);
        for (uint32_t r = 0; r < rows; ++r) {
            const uint32_t q = v->sparse.row_ptr[r];
            if (q < v->sparse.row_ptr[r + 1]) heads[q >> 5] |= 1u << (q & 31);
        }
        // CTA c's CSR entries are [row_ptr[r0], row_ptr[r1]) of its tile rows
        std::vector<uint32_t> rng(size_t(num_sms) * 2, 0);
        for (int c = 0; c < num_sms; ++c) {
            uint32_t t0, nt;
            tile_share(ntiles, num_sms, uint32_t(c), t0, nt);
            const uint32_t r0 = std::min(t0 * kTileRows, rows);
            const uint32_t r1 = std::min((t0 + nt) * kTileRows, rows);
            rng[2 * c] = v->sparse.row_ptr[r0];
            rng[2 * c + 1] = v->sparse.row_ptr[r1];
        }
        if (rec_layout) {
            L->rec = reinterpret_cast<const uint32_t*>(base + o_words);
            L->tlut = reinterpret_cast<const uint32_t*>(base + o_tlut);
            StackParams& sp = L->sp1;
            sp.counters = L->stack_counters;
            sp.gseg = L->gseg1;
            sp.gseg_cap = gseg_cap;
            StackLayerDesc& d = sp.inl[0];
            d.idx = L->rec;
            d.lut = L->tlut;
            d.row_ptr = P.row_ptr;
            d.csr = P.csr;
            d.csr_rng = L->csr_rng;
            d.csr_heads = L->csr_heads;
        }
        auto up = [&](size_t off, const void* src, size_t n) {
            return cudaMemcpy(base + off, src, n, cudaMemcpyHostToDevice);
        };
        if ((e = up(o_words, words.data(), words.size() * 4)) != cudaSuccess ||
            (tluts.size() && (e = up(o_tlut, tluts.data(), tluts.size() * 4)) != cudaSuccess) ||
            (e = up(o_lut, lut.data(), lut.size() * 2)) != cudaSuccess ||
            (e = up(o_rowptr, v->sparse.row_ptr, (size_t(rows) + 1) * 4)) != cudaSuccess ||
            (e = up(o_csr, csr.data(), csr.size() * 4)) != cudaSuccess ||
            (e = cudaMemset(base + o_counters, 0, size_t(n_rb) * 4)) != cudaSuccess ||
            (e = cudaMemset(base + o_zrp, 0, (size_t(rows) + 1) * 4)) != cudaSuccess ||
            (e = cudaMemset(base + o_scnt, 0, 2 * 4)) != cudaSuccess ||
            (e = up(o_rng, rng.data(), rng.size() * 4)) != cudaSuccess ||
            (e = up(o_heads, heads.data(), heads.size() * 4)) != cudaSuccess ||
            (e = cudaMemset(base + o_zrng, 0, size_t(num_sms) * 8)) != cudaSuccess ||
            (e = cudaMemset(base + o_x16, 0, (size_t(ng) * kGroupCols + 8) * 2)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking)) != cudaSuccess) {
            cudaFree(L->arena);
            delete L;
            return cuda_fail(e, "layer upload");
        }
    }
    *out = L;
    return DSQ_OK;
}

int dsq_cuda_layer_destroy(dsq_cuda_layer* L) {
    if (!L) return DSQ_OK;
    cudaSetDevice(L->device);
    for (auto& g : L->host_graph)
        if (g) cudaGraphExecDestroy(g);
    if (L->stream) cudaStreamDestroy(L->stream);
    if (L->x32_pin) cudaFreeHost(L->x32_pin);
    if (L->x16_pin) cudaFreeHost(L->x16_pin);
    if (L->y32_pin) cudaFreeHost(L->y32_pin);
    if (L->dense_w) cudaFree(L->dense_w);
    for (void* m : L->bs_mem)
        if (m) cudaFree(m);
    if (L->gseg2) cudaFree(L->gseg2);
    if (L->gseg4) cudaFree(L->gseg4);
    if (L->gseg8) cudaFree(L->gseg8);
    if (L->arena) cudaFree(L->arena);
    delete L;
    return DSQ_OK;
}

int dsq_cuda_layer_get_info(const dsq_cuda_layer* L, dsq_layer_info* info) {
    if (!L || !info) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    info->rows = L->rows;
    info->cols = L->cols;
    info->bits = L->bits;
    info->groups_per_row = L->groups;
    info->nnz = L->nnz;
    info->device_bytes = L->arena_bytes + (L->dense_w ? size_t(L->rows) * L->cols * 2 : 0);
    info->algorithmic_bytes = L->algorithmic_bytes;
    info->luts_exact_f16 = L->luts_exact;
    info->values_exact_f16 = L->values_exact;
    info->workers = L->n_workers;
    info->ctas = L->ctas;
    return DSQ_OK;
}

static int ensure_dense(dsq_cuda_layer* L, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(L->mu);
    if (L->dense_w) return DSQ_OK;
    CUDA_TRY(cudaMalloc(&L->dense_w, size_t(L->rows) * L->cols * 2));
    if (L->grouped)
        CUDA_TRY(launch_grouped_decode(1, L->G, L->dense_w, st));
    else if (L->rec_layout)
        CUDA_TRY(launch_decode_tiles(1, L->bits, L->rec, L->tlut, L->rows, L->cols, L->ns,
                                     L->dense_w, st));
    else
        CUDA_TRY(launch_decode(1, L->P, L->dense_w, st));
    return DSQ_OK;
}

// which kernel runs a batched product: K7 (the persistent batch-1 kernel with
// NB = 2 / 4 / 8 vectors per decoded fragment) for batch 2..4, K11 (bstream.cu:
// dense fragment map on per-warp TMA rings) for 5..16 and for batches whose x
// does not fit next to K7's ring.  DSQ_BATCH_PATH=k7 runs batch 5..8 on K7
// (NB = 8) instead, for A/B measurements.
enum class BatchRoute { k7, k11 };
static BatchRoute batch_route(const dsq_cuda_layer* L, uint32_t batch) {
    static const bool k7_to_8 = [] {
        const char* e = std::getenv("DSQ_BATCH_PATH");
        return e && !std::strcmp(e, "k7");
    }();
    const uint32_t nbk = batch == 2 ? 2u : batch <= 4 ? 4u : 8u;
    if ((batch <= 4 || (k7_to_8 && batch <= 8)) && !L->k7_batch_failed(nbk)) return BatchRoute::k7;
    return BatchRoute::k11;
}

// K11's plan for B <= 8 * nb vectors: warp ranges, segment numbering, the
// segment partials and the transposed x (caller holds L->mu)
static int ensure_bstream(dsq_cuda_layer* L, uint32_t nb) {
    if (L->bs_mem[nb - 1]) return DSQ_OK;
    static const uint32_t warps = [] {
        const char* e = std::getenv("DSQ_BS_WARPS");
        return e && std::atoi(e) == 16 ? 16u : 8u;
    }();
    const BStreamPlanHost h = bstream_plan(L->tiles, L->ns, L->bits, nb, uint32_t(L->num_sms), warps);
    const size_t smem = bstream_smem_bytes(L->bits, nb, h.max_span, h.cs, h.warps);
    if (smem > 232448 || h.phases > kBsMaxPhases)
        return fail(DSQ_E_UNSUPPORTED, "batched plan: %zu bytes of shared memory, %u phases", smem,
                    h.phases);
    auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t b_w = up(h.wdesc.size() * 4), b_s = up(h.seg_base.size() * 4),
                 b_part = up(size_t(h.nseg) * 16 * 8 * nb * 4),
                 b_xt = up(size_t(L->ns) * kSpanCols * 8 * nb * 2);
    uint8_t* m = nullptr;
    CUDA_TRY(cudaMalloc(&m, b_w + b_s + b_part + b_xt));
    BStreamDevPlan& d = L->bs[nb - 1];
    d.phases = h.phases;
    d.nseg = h.nseg;
    d.max_span = h.max_span;
    d.cs = h.cs;
    d.grid = h.grid;
    d.tiles16 = (L->tiles + 3) / 4;
    d.warps = h.warps;
    for (uint32_t k = 0; k <= h.phases; ++k) {
        d.phase_span_h[k] = h.phase_span[k];
        d.cta_pre_h[k] = h.cta_pre[k];
    }
    d.wdesc = reinterpret_cast<uint4*>(m);
    d.seg_base = reinterpret_cast<uint32_t*>(m + b_w);
    d.part = reinterpret_cast<float*>(m + b_w + b_s);
    d.xT = reinterpret_cast<uint16_t*>(m + b_w + b_s + b_part);
    cudaError_t e = cudaMemcpy(d.wdesc, h.wdesc.data(), h.wdesc.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(d.seg_base, h.seg_base.data(), h.seg_base.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(m);
        return cuda_fail(e, "batched plan upload");
    }
    L->bs_mem[nb - 1] = m;
    return DSQ_OK;
}

// batched products on K11 (bstream.cu): x [batch][cols]
// fp16, y [batch][rows]
static int gemv_batch(dsq_cuda_layer* L, int kernel, const void* x, int x_dtype, void* y,
                      int y_dtype, uint32_t batch, cudaStream_t st, uint32_t x_stride,
                      uint32_t y_stride) {
    if (kernel < DSQ_KERNEL_LUT || kernel > DSQ_KERNEL_FUSED)
        return fail(DSQ_E_UNSUPPORTED, "batched products: LUT, CSR or FUSED kernels");
    if (!L->rec_layout)
        return fail(DSQ_E_UNSUPPORTED, "batched products need bits 3 or 4 (got %u)", L->bits);
    if (x_dtype != DSQ_F16) return fail(DSQ_E_INVALID_ARGUMENT, "batched x must be F16");
    if ((reinterpret_cast<uintptr_t>(x) & 15u) || (x_stride % 8))
        return fail(DSQ_E_INVALID_ARGUMENT, "batched x rows must be 16-byte aligned (stride %% 8 == 0)");
    if (y_dtype != DSQ_F32 && y_dtype != DSQ_F16)
        return fail(DSQ_E_INVALID_ARGUMENT, "y dtype must be F32 or F16");
    const int mode = kernel == DSQ_KERNEL_LUT ? 0 : kernel == DSQ_KERNEL_CSR ? 1 : 2;
    const uint32_t nb = batch > 8 ? 2u : 1u;
    {
        std::lock_guard<std::mutex> lk(L->mu);
        const int rc = ensure_bstream(L, nb);
        if (rc) return rc;
    }
    CUDA_TRY(launch_bstream(L->bits, nb, L->bs[nb - 1], L->rec, L->tlut, L->P.row_ptr, L->P.csr,
                            L->rows, L->cols, L->ns, L->tiles, static_cast<const uint16_t*>(x),
                            x_stride, batch, y, y_stride, y_dtype == DSQ_F16, mode, st));
    return DSQ_OK;
}

// x_stride / y_stride: elements between the batch's vectors (0: cols / rows)
static int gemv_impl(const dsq_cuda_layer* Lc, int kernel, const void* x, int x_dtype, void* y,
                     int y_dtype, uint32_t batch, cudaStream_t st, bool pdl,
                     uint32_t x_stride = 0, uint32_t y_stride = 0) {
    auto* L = const_cast<dsq_cuda_layer*>(Lc);
    if (!L || !x || !y) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    if (!x_stride) x_stride = L->cols;
    if (!y_stride) y_stride = L->rows;
    if (batch < 1 || batch > 16) return fail(DSQ_E_INVALID_ARGUMENT, "batch must be 1..16");
    if (L->grouped && kernel != DSQ_KERNEL_REFERENCE) {
        // grouped LUTs: one grouped_gemv launch per vector
        if (kernel < DSQ_KERNEL_LUT || kernel > DSQ_KERNEL_FUSED)
            return fail(DSQ_E_INVALID_ARGUMENT, "unknown kernel %d", kernel);
        if (y_dtype != DSQ_F32 && y_dtype != DSQ_F16)
            return fail(DSQ_E_INVALID_ARGUMENT, "y dtype must be F32 or F16");
        if (x_dtype == DSQ_F32 && batch != 1)
            return fail(DSQ_E_INVALID_ARGUMENT, "batched x must be F16");
        const int mode = kernel == DSQ_KERNEL_LUT ? 0 : kernel == DSQ_KERNEL_CSR ? 1 : 2;
        const size_t ysz = y_dtype == DSQ_F16 ? 2 : 4;
        for (uint32_t b = 0; b < batch; ++b) {
            const uint16_t* xb;
            if (x_dtype == DSQ_F32) {
                CUDA_TRY(launch_f32_to_f16(static_cast<const float*>(x), L->x16, L->cols, st, pdl));
                xb = L->x16;
            } else if (x_dtype == DSQ_F16) {
                xb = static_cast<const uint16_t*>(x) + size_t(b) * x_stride;
            } else {
                return fail(DSQ_E_INVALID_ARGUMENT, "x dtype must be F32 or F16");
            }
            CUDA_TRY(launch_grouped(mode, L->G, xb, static_cast<uint8_t*>(y) + size_t(b) * y_stride * ysz,
                                    y_dtype == DSQ_F16, st, pdl));
        }
        return DSQ_OK;
    }
    if (L->grouped && batch > 1)
        return fail(DSQ_E_UNSUPPORTED, "grouped LUTs: batched reference kernel");
    const uint32_t nbk = batch == 2 ? 2u : batch <= 4 ? 4u : 8u;
    if (batch >= 2 && batch <= 8 && L->rec_layout && batch_route(L, batch) == BatchRoute::k7 &&
        (kernel == DSQ_KERNEL_LUT || kernel == DSQ_KERNEL_FUSED) &&
        x_dtype == DSQ_F16 && (y_dtype == DSQ_F32 || y_dtype == DSQ_F16) &&
        !(reinterpret_cast<uintptr_t>(x) & 15u) && x_stride % 8 == 0) {
        // K7 with 2 or 4 activation vectors in one launch: all share every
        // decoded weight fragment (vectors 0/1 in the HMMA B columns 0..3 /
        // 4..7, vectors 2/3 in a second HMMA on the same A fragment)
        const uint32_t nb = nbk;
        StackParams& spb = nb == 2 ? L->sp2 : nb == 4 ? L->sp4 : L->sp8;
        {
            std::lock_guard<std::mutex> lk(L->mu);
            bool& ready = nb == 2 ? L->sp2_ready : nb == 4 ? L->sp4_ready : L->sp8_ready;
            float*& gbuf = nb == 2 ? L->gseg2 : nb == 4 ? L->gseg4 : L->gseg8;
            if (!ready) {
                uint32_t gcap = 0;
                StackPlanLayer pl{L->rows, L->cols, L->tiles, L->ns,
                                  max_nnz_per_cta(L->row_ptr_host, L->rows, L->num_sms)};
                int prc = plan_stack(&pl, 1, L->num_sms, L->bits, spb, gcap, nb);
                if (prc == DSQ_E_UNSUPPORTED) {  // the x vectors do not fit: the K11 path
                    (nb == 2 ? L->sp2_failed : nb == 4 ? L->sp4_failed : L->sp8_failed) = true;
                    goto batched_k11;
                }
                if (prc) return prc;
                if (gcap)
                    CUDA_TRY(cudaMalloc(&gbuf, size_t(L->num_sms) * 2 * nb * gcap * 4 + 4));
                StackParams& q = spb;
                const StackLayerDesc& d1 = L->sp1.inl[0];
                StackLayerDesc& d = q.inl[0];
                d.idx = d1.idx;
                d.lut = d1.lut;
                d.row_ptr = d1.row_ptr;
                d.csr = d1.csr;
                d.csr_rng = d1.csr_rng;
                d.csr_heads = d1.csr_heads;
                d.dep = kNoDep;
                d.reduce_ord = kNoDep;
                q.counters = L->sp1.counters;
                q.gseg = gbuf;
                q.gseg_cap = gcap;
                ready = true;
            }
        }
        StackParams sp = spb;
        sp.nvec = batch;
        StackLayerDesc& d = sp.inl[0];
        d.x = static_cast<const uint16_t*>(x);
        d.y = y;
        d.y_f16 = y_dtype == DSQ_F16 ? 1u : 0u;
        if (kernel == DSQ_KERNEL_LUT) {  // LUT part only: empty CSR
            d.row_ptr = L->zero_rp;
            d.csr_rng = L->zero_rng;
        }
        sp.x_bstride = x_stride;
        sp.y_bstride = y_stride;
        sp.n_layers = 1;
        sp.layers = nullptr;
        CUDA_TRY(launch_stack(sp, st, pdl));
        return DSQ_OK;
    }
batched_k11:
    if (batch > 1)
        return gemv_batch(L, kernel, x, x_dtype, y, y_dtype, batch, st, x_stride, y_stride);
    if (kernel < DSQ_KERNEL_LUT || kernel > DSQ_KERNEL_REFERENCE)
        return fail(DSQ_E_INVALID_ARGUMENT, "unknown kernel %d", kernel);
    if (y_dtype != DSQ_F32 && y_dtype != DSQ_F16)
        return fail(DSQ_E_INVALID_ARGUMENT, "y dtype must be F32 or F16");
    const uint16_t* x16;
    if (x_dtype == DSQ_F32) {
        CUDA_TRY(launch_f32_to_f16(static_cast<const float*>(x), L->x16, L->cols, st, pdl));
        x16 = L->x16;
    } else if (x_dtype == DSQ_F16) {
        if (reinterpret_cast<uintptr_t>(x) & 15u)
            return fail(DSQ_E_INVALID_ARGUMENT, "fp16 x must be 16-byte aligned");
        x16 = static_cast<const uint16_t*>(x);
    } else {
        return fail(DSQ_E_INVALID_ARGUMENT, "x dtype must be F32 or F16");
    }
    const bool yh = y_dtype == DSQ_F16;
    if (kernel == DSQ_KERNEL_REFERENCE) {
        int rc = ensure_dense(L, st);
        if (rc) return rc;
        CUDA_TRY(launch_dense(L->dense_w, L->rows, L->cols, x16, y, yh, L->num_sms, st, pdl));
        return DSQ_OK;
    }
    const int mode = kernel == DSQ_KERNEL_LUT ? 0 : kernel == DSQ_KERNEL_CSR ? 1 : 2;
    if (L->rec_layout && mode != 1) {
        // K7 persistent kernel, one layer carried inline in the launch params
        StackParams sp = L->sp1;
        StackLayerDesc& d = sp.inl[0];
        d.x = x16;
        d.y = y;
        d.y_f16 = yh ? 1u : 0u;
        if (mode == 0) {  // LUT part only: empty CSR
            d.row_ptr = L->zero_rp;
            d.csr_rng = L->zero_rng;
        }
        sp.n_layers = 1;
        sp.layers = nullptr;
        CUDA_TRY(launch_stack(sp, st, pdl));
        return DSQ_OK;
    }
    CUDA_TRY(launch_fused(mode, L->P, L->W, x16, y, yh, L->ctas, st, pdl));
    return DSQ_OK;
}

int dsq_cuda_gemv(const dsq_cuda_layer* L, int kernel, const void* x, int x_dtype, void* y,
                  int y_dtype, uint32_t batch, void* stream) {
    if (L) cudaSetDevice(L->device);
    return gemv_impl(L, kernel, x, x_dtype, y, y_dtype, batch, static_cast<cudaStream_t>(stream),
                     true);
}

int dsq_cuda_lut_gemv(const dsq_cuda_layer* L, const void* x, int xd, void* y, int yd,
                      uint32_t batch, void* stream) {
    return dsq_cuda_gemv(L, DSQ_KERNEL_LUT, x, xd, y, yd, batch, stream);
}
int dsq_cuda_csr_gemv(const dsq_cuda_layer* L, const void* x, int xd, void* y, int yd,
                      uint32_t batch, void* stream) {
    return dsq_cuda_gemv(L, DSQ_KERNEL_CSR, x, xd, y, yd, batch, stream);
}
int dsq_cuda_fused_gemv(const dsq_cuda_layer* L, const void* x, int xd, void* y, int yd,
                        uint32_t batch, void* stream) {
    return dsq_cuda_gemv(L, DSQ_KERNEL_FUSED, x, xd, y, yd, batch, stream);
}

int dsq_cuda_dense_gemv(const uint16_t* w, uint32_t rows, uint32_t cols, const void* x,
                        int x_dtype, void* y, int y_dtype, void* stream) {
    if (!w || !x || !y) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    if (rows < 1 || cols < 1) return fail(DSQ_E_EMPTY_DIMENSION, "dense: empty dims");
    if (x_dtype != DSQ_F16) return fail(DSQ_E_INVALID_ARGUMENT, "dense: x must be F16");
    if (y_dtype != DSQ_F32 && y_dtype != DSQ_F16)
        return fail(DSQ_E_INVALID_ARGUMENT, "y dtype must be F32 or F16");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    int rc = query_num_sms(dev, &sms);
    if (rc) return rc;
    CUDA_TRY(launch_dense(w, rows, cols, static_cast<const uint16_t*>(x), y, y_dtype == DSQ_F16,
                          sms, static_cast<cudaStream_t>(stream), true));
    return DSQ_OK;
}

// host-side conversions of the reference-signature call: fp32 -> fp16
// (round to nearest even, like __float2half_rn) with F16C, fp32 -> fp64 with
// AVX; scalar fallbacks on CPUs without them
__attribute__((target("avx,f16c"))) static void f32_to_f16_f16c(const float* in, uint16_t* out,
                                                                size_t n) {
    size_t i = 0;
    for (; i + 8 <= n; i += 8)
        _mm_storeu_si128(reinterpret_cast<__m128i*>(out + i),
                         _mm256_cvtps_ph(_mm256_loadu_ps(in + i), _MM_FROUND_TO_NEAREST_INT));
    for (; i < n; ++i) out[i] = f32_to_f16(in[i]);
}
__attribute__((target("avx"))) static void f32_to_f64_avx(const float* in, double* out,
                                                          size_t n) {
    size_t i = 0;
    for (; i + 4 <= n; i += 4) _mm256_storeu_pd(out + i, _mm256_cvtps_pd(_mm_loadu_ps(in + i)));
    for (; i < n; ++i) out[i] = double(in[i]);
}
static void host_x_to_f16(const float* in, uint16_t* out, size_t n) {
    static const bool f16c = __builtin_cpu_supports("f16c") && __builtin_cpu_supports("avx");
    if (f16c) {
        f32_to_f16_f16c(in, out, n);
    } else {
        for (size_t i = 0; i < n; ++i) out[i] = f32_to_f16(in[i]);
    }
}
static void host_y_to_f64(const float* in, double* out, size_t n) {
    static const bool avx = __builtin_cpu_supports("avx");
    if (avx) {
        f32_to_f64_avx(in, out, n);
    } else {
        for (size_t i = 0; i < n; ++i) out[i] = double(in[i]);
    }
}

// The reference-signature product (fp32 host x -> fp64 host y): x is
// converted to fp16 on the host straight into pinned, device-mapped staging;
// one captured CUDA graph per kernel replays "pinned x16 -> device x16 (one
// small PDL copy kernel) -> the product, y written as fp32 straight into
// pinned, device-mapped host memory"; then one stream synchronisation and a
// vectorised fp64 widen.  (The x / y buffers are the layer's own, so the
// graph is captured once and replayed.)
int dsq_cuda_matvec_host(const dsq_cuda_layer* Lc, int kernel, const float* x_host,
                         double* y_host) {
    auto* L = const_cast<dsq_cuda_layer*>(Lc);
    if (!L || !x_host || !y_host) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    if (kernel < DSQ_KERNEL_LUT || kernel > DSQ_KERNEL_REFERENCE)
        return fail(DSQ_E_INVALID_ARGUMENT, "unknown kernel %d", kernel);
    cudaSetDevice(L->device);
    std::lock_guard<std::mutex> lk(L->host_mu);
    const size_t x16_bytes = (size_t(L->cols) * 2 + 15) / 16 * 16;
    if (!L->x16_pin) {
        const unsigned fl = cudaHostAllocMapped | cudaHostAllocPortable;
        cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&L->x16_pin), x16_bytes, fl);
        if (e == cudaSuccess && !L->y32_pin)
            e = cudaHostAlloc(reinterpret_cast<void**>(&L->y32_pin), size_t(L->rows) * 4, fl);
        if (e == cudaSuccess)
            e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&L->x16_map), L->x16_pin, 0);
        if (e == cudaSuccess)
            e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&L->y32_map), L->y32_pin, 0);
        if (e != cudaSuccess) {
            if (L->x16_pin) cudaFreeHost(L->x16_pin);
            if (L->y32_pin) cudaFreeHost(L->y32_pin);
            L->x16_pin = nullptr;
            L->y32_pin = nullptr;
            L->x16_map = nullptr;
            L->y32_map = nullptr;
            return cuda_fail(e, "host-API staging");
        }
        std::memset(L->x16_pin, 0, x16_bytes);
    }
    cudaGraphExec_t& g = L->host_graph[kernel];
    if (!g) {
        if (kernel == DSQ_KERNEL_REFERENCE) {  // allocation must precede the capture
            int rc = ensure_dense(L, L->stream);
            if (rc) return rc;
            CUDA_TRY(cudaStreamSynchronize(L->stream));
        }
        cudaGraph_t graph = nullptr;
        CUDA_TRY(cudaStreamBeginCapture(L->stream, cudaStreamCaptureModeThreadLocal));
        cudaError_t e = launch_upload_x(L->x16_map, L->x16, x16_bytes, L->stream);
        int rc = e == cudaSuccess ? gemv_impl(L, kernel, L->x16, DSQ_F16, L->y32_map, DSQ_F32, 1,
                                              L->stream, true)
                                  : DSQ_OK;
        cudaError_t e2 = cudaStreamEndCapture(L->stream, &graph);
        if (e != cudaSuccess) return cuda_fail(e, "host-API graph capture (upload)");
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (e2 != cudaSuccess) return cuda_fail(e2, "host-API graph capture");
        e = cudaGraphInstantiate(&g, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            g = nullptr;
            return cuda_fail(e, "host-API graph instantiate");
        }
    }
    host_x_to_f16(x_host, L->x16_pin, L->cols);
    std::atomic_thread_fence(std::memory_order_seq_cst);
    CUDA_TRY(cudaGraphLaunch(g, L->stream));
    CUDA_TRY(cudaStreamSynchronize(L->stream));
    host_y_to_f64(L->y32_pin, y_host, L->rows);
    return DSQ_OK;
}

int dsq_cuda_unpack(const dsq_cuda_layer* L, uint16_t* assign_dev, void* stream) {
    if (!L || !assign_dev) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    cudaSetDevice(L->device);
    if (L->grouped)
        CUDA_TRY(launch_grouped_decode(0, L->G, assign_dev, static_cast<cudaStream_t>(stream)));
    else if (L->rec_layout)
        CUDA_TRY(launch_decode_tiles(0, L->bits, L->rec, L->tlut, L->rows, L->cols, L->ns,
                                     assign_dev, static_cast<cudaStream_t>(stream)));
    else
        CUDA_TRY(launch_decode(0, L->P, assign_dev, static_cast<cudaStream_t>(stream)));
    return DSQ_OK;
}

int dsq_cuda_dequant(const dsq_cuda_layer* L, void* w_dev, int out_dtype, void* stream) {
    if (!L || !w_dev) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    if (out_dtype != DSQ_F16 && out_dtype != DSQ_F32)
        return fail(DSQ_E_INVALID_ARGUMENT, "dequant: out dtype must be F16 or F32");
    cudaSetDevice(L->device);
    const int mode = out_dtype == DSQ_F16 ? 1 : 2;
    if (L->grouped)
        CUDA_TRY(launch_grouped_decode(mode, L->G, w_dev, static_cast<cudaStream_t>(stream)));
    else if (L->rec_layout)
        CUDA_TRY(launch_decode_tiles(mode, L->bits, L->rec, L->tlut, L->rows, L->cols, L->ns,
                                     w_dev, static_cast<cudaStream_t>(stream)));
    else
        CUDA_TRY(launch_decode(mode, L->P, w_dev, static_cast<cudaStream_t>(stream)));
    return DSQ_OK;
}

int dsq_cuda_dump_frags(const dsq_cuda_layer* L, uint16_t* w_dev, void* stream) {
    if (!L || !w_dev) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    if (!L->rec_layout)
        return fail(DSQ_E_UNSUPPORTED, "dump_frags: only the 3/4-bit tile layout has HMMA fragments");
    cudaSetDevice(L->device);
    CUDA_TRY(launch_dump_frags(L->bits, L->rec, L->tlut, L->rows, L->cols, L->tiles, L->ns, w_dev,
                               static_cast<cudaStream_t>(stream)));
    return DSQ_OK;
}

// ---- reference-signature host products (the sqz:: C++ drop-in functions) ----

int dsq_cuda_dequantize_layer(const dsq_cuda_layer* L, float* w_dev, void* stream) {
    if (!L || !w_dev) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    cudaSetDevice(L->device);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (L->grouped)
        CUDA_TRY(launch_grouped_decode(2, L->G, w_dev, st));
    else if (L->rec_layout)
        CUDA_TRY(launch_decode_tiles(2, L->bits, L->rec, L->tlut, L->rows, L->cols, L->ns, w_dev,
                                     st));
    else
        CUDA_TRY(launch_decode(2, L->P, w_dev, st));
    if (L->nnz)
        CUDA_TRY(launch_apply_deltas(L->P.row_ptr, L->P.csr, L->P.lut, 1u << L->bits, L->groups,
                                     L->cols / L->groups, L->rows, L->cols, w_dev, st));
    return DSQ_OK;
}

int dsq_cuda_dequantize_layer_host(const dsq_cuda_layer* Lc, float* w_host) {
    auto* L = const_cast<dsq_cuda_layer*>(Lc);
    if (!L || !w_host) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    cudaSetDevice(L->device);
    std::lock_guard<std::mutex> lk(L->host_mu);
    const size_t bytes = size_t(L->rows) * L->cols * 4;
    float* w = nullptr;
    CUDA_TRY(cudaMalloc(&w, bytes));
    int rc = dsq_cuda_dequantize_layer(L, w, L->stream);
    cudaError_t e = rc ? cudaSuccess : cudaMemcpyAsync(w_host, w, bytes, cudaMemcpyDeviceToHost,
                                                       L->stream);
    if (!rc && e == cudaSuccess) e = cudaStreamSynchronize(L->stream);
    cudaFree(w);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "dequantize_layer");
    return DSQ_OK;
}

int dsq_cuda_dense_matvec_host(const float* m, uint32_t rows, uint32_t cols, const float* x,
                               double* y, int device) {
    if (!m || !x || !y) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    if (rows < 1 || cols < 1) return fail(DSQ_E_EMPTY_DIMENSION, "dense: empty dims");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(DSQ_E_NO_DEVICE, "no CUDA device visible");
    if (device < 0 || device >= ndev) return fail(DSQ_E_NO_DEVICE, "bad device %d", device);
    CUDA_TRY(cudaSetDevice(device));
    int sms = 0;
    int rc = query_num_sms(device, &sms);
    if (rc) return rc;
    const size_t wb = size_t(rows) * cols * 4;
    uint8_t* buf = nullptr;
    CUDA_TRY(cudaMalloc(&buf, wb + size_t(cols) * 4 + size_t(rows) * 8 + 512));
    float* dw = reinterpret_cast<float*>(buf);
    float* dx = reinterpret_cast<float*>(buf + ((wb + 255) & ~size_t(255)));
    double* dy = reinterpret_cast<double*>(buf + ((wb + 255) & ~size_t(255)) +
                                           ((size_t(cols) * 4 + 255) & ~size_t(255)));
    cudaError_t e = cudaMemcpy(dw, m, wb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dx, x, size_t(cols) * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_dense_f32(dw, rows, cols, dx, dy, sms, nullptr);
    if (e == cudaSuccess) e = cudaMemcpy(y, dy, size_t(rows) * 8, cudaMemcpyDeviceToHost);
    cudaFree(buf);
    if (e != cudaSuccess) return cuda_fail(e, "dense_matvec");
    return DSQ_OK;
}

// one-shot products of a bare PackedDense / CsrMatrix: a transient layer
// whose other part is empty (no CSR entries / an all-zero 1-bit LUT part)
int dsq_cuda_packed_matvec_host(const dsq_packed_view* p, const float* x, double* y,
                                int device) {
    if (!p || !x || !y) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    std::vector<uint32_t> zrp(size_t(p->rows) + 1, 0);
    dsq_layer_view v{};
    v.name = "packed";
    v.rows = p->rows;
    v.cols = p->cols;
    v.packed = *p;
    v.sparse.rows = p->rows;
    v.sparse.cols = p->cols;
    v.sparse.row_ptr = zrp.data();
    dsq_cuda_layer* L = nullptr;
    int rc = dsq_cuda_layer_create(&v, device, &L);
    if (rc) return rc;
    rc = dsq_cuda_matvec_host(L, DSQ_KERNEL_LUT, x, y);
    dsq_cuda_layer_destroy(L);
    return rc;
}

int dsq_cuda_csr_matvec_host(const dsq_csr_view* s, const float* x, double* y, int device) {
    if (!s || !x || !y) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    if (s->cols >= 65536u) return fail(DSQ_E_DIMENSION_OVERFLOW, "csr: cols must be < 65536");
    if (s->rows < 1 || s->cols < 1) return fail(DSQ_E_EMPTY_DIMENSION, "csr: empty dims");
    std::vector<float> zl(size_t(s->rows) * 2, 0.f);
    std::vector<uint8_t> zp(size_t(s->rows) * row_stride(s->cols, 1), 0);
    dsq_layer_view v{};
    v.name = "csr";
    v.rows = s->rows;
    v.cols = s->cols;
    v.packed.bits = 1;
    v.packed.rows = s->rows;
    v.packed.cols = s->cols;
    v.packed.groups_per_row = 1;
    v.packed.luts_f32 = zl.data();
    v.packed.payload = zp.data();
    v.packed.payload_len = zp.size();
    v.sparse = *s;
    dsq_cuda_layer* L = nullptr;
    int rc = dsq_cuda_layer_create(&v, device, &L);
    if (rc) return rc;
    rc = dsq_cuda_matvec_host(L, DSQ_KERNEL_CSR, x, y);
    dsq_cuda_layer_destroy(L);
    return rc;
}

struct dsq_cuda_tp {
    int device = 0;
    uint32_t world = 1, rank = 0, max_rows = 0, max_grid = 0;
    void* buf = nullptr;           // recv [2][world][max_rows] {fp32, u32 tag} + flags [max_grid] u32
    size_t recv_bytes = 0;
    uint64_t base = 0;             // reduce ordinals completed by earlier launches
    void* peer_base[8] = {};       // mapped peer buffers (own: buf)
    bool peer_ipc[8] = {};
};

// a stack step run as its own product launch (the sequential form)
struct StackSeqStep {
    const dsq_cuda_layer* layer;
    const void* x;
    void* y;
    uint32_t x_stride, y_stride;
};

struct dsq_cuda_stack {
    int device = 0;
    uint32_t n = 0;
    uint32_t n_reduce = 0;
    // sequential form: batches the persistent kernel cannot hold (5..16, or
    // x vectors that do not fit next to the ring) run layer by layer through
    // the batched product kernels, back to back under PDL
    bool seq = false;
    uint32_t batch = 1, y_dtype = DSQ_F16, launches = 1;
    std::vector<StackSeqStep> steps;
    // the sequential form's launches captured once (after one eager run has
    // created the layers' batched plans) and replayed as one graph launch
    cudaStream_t seq_capture = nullptr;
    cudaGraphExec_t seq_graph = nullptr;
    uint32_t seq_runs = 0;
    // serving loop (dsq_cuda_serve_*): device [gate n][notify n][flag][err],
    // pinned host [host_done][doorbell] and the x staging buffer
    uint32_t* serve_dev = nullptr;
    uint32_t* serve_pin = nullptr;
    void* serve_x_pin = nullptr;  // pinned, device-mapped x staging
    void* serve_ll_pin = nullptr;  // pinned, device-mapped tagged output words
    size_t serve_ll_cap = 0;
    uint32_t* serve_y_host = nullptr;  // the caller's output buffer (serve_begin)
    size_t serve_x_cap = 0, serve_x_bytes = 0;
    size_t serve_y_cap = 0;  // bytes of the smallest notify layer's y (0: unaligned)
    const void* serve_x_ptr = nullptr;  // the gated layers' (common) x buffer
    uint32_t serve_x_cols = 0;          // their (common) column count
    cudaStream_t serve_stream = nullptr;
    uint32_t serve_steps = 0, serve_k = 0;
    bool serving = false;
    dsq_cuda_tp* tp = nullptr;
    StackParams sp{};
    void* arena = nullptr;
    unsigned long long* trace = nullptr;  // DSQ_STACK_TRACE=1: per-CTA layer timeline
};

static int stack_create_impl(dsq_cuda_layer* const* layers, uint32_t n, const int32_t* deps,
                             const void* const* xs, void* const* ys, int y_dtype,
                             const uint8_t* reduce, dsq_cuda_tp* tp, uint32_t grid,
                             dsq_cuda_stack** out, uint32_t batch = 1, uint32_t x_bstride = 0,
                             uint32_t y_bstride = 0) {
    if (!out || !layers || !deps || !xs || !ys || n == 0)
        return fail(DSQ_E_INVALID_ARGUMENT, "stack: null argument or empty stack");
    *out = nullptr;
    if (batch < 1 || batch > 16)
        return fail(DSQ_E_INVALID_ARGUMENT, "stack: batch must be 1..16");
    const uint32_t nbatch = batch == 1 ? 1u : batch == 2 ? 2u : 4u;
    if (batch > 1) {
        if (tp) return fail(DSQ_E_UNSUPPORTED, "stack: batched stacks are single-GPU");
        if (x_bstride % 8 || y_bstride % 8)
            return fail(DSQ_E_INVALID_ARGUMENT, "stack: batch strides must be multiples of 8");
        for (uint32_t i = 0; i < n; ++i) {
            if (!layers[i]) break;
            if (layers[i]->rows > y_bstride)
                return fail(DSQ_E_INVALID_ARGUMENT, "stack: y batch stride < rows of layer %u", i);
            if (deps[i] < 0 && layers[i]->cols > x_bstride)
                return fail(DSQ_E_INVALID_ARGUMENT, "stack: x batch stride < cols of layer %u", i);
        }
    }
    if (y_dtype != DSQ_F32 && y_dtype != DSQ_F16)
        return fail(DSQ_E_INVALID_ARGUMENT, "stack: y dtype must be F32 or F16");
    const dsq_cuda_layer* L0 = layers[0];
    if (!L0) return fail(DSQ_E_INVALID_ARGUMENT, "stack: null layer");
    const int G = grid ? int(grid) : L0->num_sms;
    if (G < 1 || G > L0->num_sms)
        return fail(DSQ_E_INVALID_ARGUMENT, "stack: grid must be 1..%d CTAs", L0->num_sms);
    if (tp && (tp->device != L0->device || uint32_t(G) > tp->max_grid))
        return fail(DSQ_E_INVALID_ARGUMENT, "stack: TP context device / grid mismatch");
    std::vector<StackPlanLayer> pl(n);
    uint32_t n_reduce = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const dsq_cuda_layer* L = layers[i];
        if (!L) return fail(DSQ_E_INVALID_ARGUMENT, "stack: null layer %u", i);
        if (!L->rec_layout || L->bits != L0->bits)
            return fail(DSQ_E_UNSUPPORTED, "stack: layers must all be 3-bit or all 4-bit");
        if (L->device != L0->device)
            return fail(DSQ_E_INVALID_ARGUMENT, "stack: layers on different devices");
        if (deps[i] >= 0) {
            if (uint32_t(deps[i]) >= i)
                return fail(DSQ_E_INVALID_ARGUMENT, "stack: deps[%u] must precede it", i);
            if (layers[deps[i]]->rows != L->cols)
                return fail(DSQ_E_SHAPE_MISMATCH, "stack: layer %u cols != rows of its input", i);
            if (y_dtype != DSQ_F16)
                return fail(DSQ_E_INVALID_ARGUMENT, "stack: chained layers need F16 outputs");
        } else if (!xs[i] || (reinterpret_cast<uintptr_t>(xs[i]) & 15u)) {
            return fail(DSQ_E_INVALID_ARGUMENT, "stack: x %u must be a 16-byte aligned fp16 buffer", i);
        }
        if (!ys[i]) return fail(DSQ_E_INVALID_ARGUMENT, "stack: null y %u", i);
        if (reduce && reduce[i]) {
            if (!tp) return fail(DSQ_E_INVALID_ARGUMENT, "stack: reduce layer %u without TP context", i);
            if (L->rows > tp->max_rows)
                return fail(DSQ_E_SHAPE_MISMATCH, "stack: reduce layer %u rows > TP max_rows", i);
            ++n_reduce;
        }
        pl[i] = StackPlanLayer{L->rows, L->cols, L->tiles, L->ns,
                               max_nnz_per_cta(L->row_ptr_host, L->rows, G)};
    }
    CUDA_TRY(cudaSetDevice(L0->device));
    auto* S = new dsq_cuda_stack;
    S->device = L0->device;
    S->n = n;
    S->n_reduce = n_reduce;
    S->tp = tp;
    S->batch = batch;
    S->y_dtype = uint32_t(y_dtype);
    uint32_t gseg_cap = 0;
    int rc = batch > 4 ? DSQ_E_UNSUPPORTED : plan_stack(pl.data(), n, G, L0->bits, S->sp, gseg_cap, nbatch);
    if (rc == DSQ_E_UNSUPPORTED && !tp && !grid) {
        // too many vectors for the persistent kernel: one product launch per layer
        S->seq = true;
        S->launches = 0;
        for (uint32_t i = 0; i < n; ++i) {
            const bool chained = deps[i] >= 0;
            S->steps.push_back(StackSeqStep{layers[i], chained ? ys[deps[i]] : xs[i], ys[i],
                                            chained ? y_bstride : x_bstride, y_bstride});
        }
        *out = S;
        return DSQ_OK;
    }
    if (rc) {
        delete S;
        return rc;
    }
    // per-(layer, CTA) CSR entry ranges for this grid
    std::vector<uint32_t> rng(size_t(n) * G * 2);
    for (uint32_t i = 0; i < n; ++i) {
        const dsq_cuda_layer* L = layers[i];
        for (int c = 0; c < G; ++c) {
            uint32_t t0, nt;
            tile_share(L->tiles, G, uint32_t(c), t0, nt);
            const uint32_t r0 = std::min(t0 * kTileRows, L->rows);
            const uint32_t r1 = std::min((t0 + nt) * kTileRows, L->rows);
            rng[(size_t(i) * G + c) * 2] = L->row_ptr_host[r0];
            rng[(size_t(i) * G + c) * 2 + 1] = L->row_ptr_host[r1];
        }
    }
    const size_t tb = (size_t(n) * sizeof(StackLayerDesc) + 255) & ~size_t(255);
    const size_t cb = ((size_t(n) + 1) * 4 + 255) & ~size_t(255);
    const size_t rb = (rng.size() * 4 + 255) & ~size_t(255);
    const size_t gb = size_t(G) * 2 * nbatch * gseg_cap * 4 + 4;
    cudaError_t e = cudaMalloc(&S->arena, tb + cb + rb + gb);
    if (e != cudaSuccess) {
        delete S;
        return cuda_fail(e, "cudaMalloc(stack)");
    }
    uint8_t* base = static_cast<uint8_t*>(S->arena);
    const uint32_t* drng = reinterpret_cast<const uint32_t*>(base + tb + cb);
    std::vector<StackLayerDesc> descs(n);
    uint32_t ord = 0;
    for (uint32_t i = 0; i < n; ++i) {
        StackLayerDesc& d = descs[i];
        fill_desc(d, pl[i], S->sp.slot_bytes, L0->bits, G, S->sp.consumers);
        const dsq_cuda_layer* L = layers[i];
        d.idx = L->rec;
        d.lut = L->tlut;
        d.row_ptr = L->P.row_ptr;
        d.csr = L->P.csr;
        d.csr_rng = drng + size_t(i) * G * 2;
        d.csr_heads = L->csr_heads;
        d.dep = deps[i] >= 0 ? uint32_t(deps[i]) : kNoDep;
        d.x = deps[i] >= 0 ? static_cast<const uint16_t*>(ys[deps[i]])
                           : static_cast<const uint16_t*>(xs[i]);
        d.y = ys[i];
        d.y_f16 = y_dtype == DSQ_F16 ? 1u : 0u;
        d.reduce_ord = (reduce && reduce[i]) ? ord++ : kNoDep;
        if (i < kInlineLayers) S->sp.inl[i] = d;
    }
    if ((e = cudaMemcpy(base, descs.data(), n * sizeof(StackLayerDesc), cudaMemcpyHostToDevice)) !=
            cudaSuccess ||
        (e = cudaMemset(base + tb, 0, cb)) != cudaSuccess ||
        (e = cudaMemcpy(base + tb + cb, rng.data(), rng.size() * 4, cudaMemcpyHostToDevice)) !=
            cudaSuccess) {
        cudaFree(S->arena);
        delete S;
        return cuda_fail(e, "stack upload");
    }
    S->sp.layers = reinterpret_cast<const StackLayerDesc*>(base);
    S->sp.counters = reinterpret_cast<uint32_t*>(base + tb);
    S->sp.gseg = reinterpret_cast<float*>(base + tb + cb + rb);
    S->sp.gseg_cap = gseg_cap;
    S->sp.nvec = batch;
    S->sp.x_bstride = x_bstride;
    S->sp.y_bstride = y_bstride;
    S->sp.n_layers = n;
    S->sp.tp_world = tp ? tp->world : 1;
    S->sp.tp_rank = tp ? tp->rank : 0;
    S->sp.tp_max_rows = tp ? tp->max_rows : 0;
    if (tp) {
        S->sp.tp_recv = static_cast<unsigned long long*>(tp->buf);
        S->sp.tp_flags = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(tp->buf) + tp->recv_bytes);
        for (uint32_t k = 0; k < tp->world; ++k)
            S->sp.tp_peer_recv[k] = static_cast<unsigned long long*>(tp->peer_base[k]);
    }
    S->sp.trace = nullptr;
    S->sp.dbg = 0;
    if (const char* t = std::getenv("DSQ_STACK_DBG")) S->sp.dbg = uint32_t(atoi(t));
    if (const char* t = std::getenv("DSQ_STACK_TRACE")) {
        if (t[0] == '1') {
            const size_t tbytes =
                std::max<size_t>(size_t(S->sp.grid) * n * kTrSlots, size_t(S->sp.grid) * 24 * 5) * 8;
            if (cudaMalloc(&S->trace, tbytes) == cudaSuccess) {
                cudaMemset(S->trace, 0, tbytes);
                S->sp.trace = S->trace;
            }
        }
    }
    *out = S;
    return DSQ_OK;
}

int dsq_cuda_stack_create(dsq_cuda_layer* const* layers, uint32_t n, const int32_t* deps,
                          const void* const* xs, void* const* ys, int y_dtype,
                          dsq_cuda_stack** out) {
    return stack_create_impl(layers, n, deps, xs, ys, y_dtype, nullptr, nullptr, 0, out);
}

int dsq_cuda_stack_create_tp(dsq_cuda_layer* const* layers, uint32_t n, const int32_t* deps,
                             const void* const* xs, void* const* ys, int y_dtype,
                             const uint8_t* reduce, dsq_cuda_tp* tp, uint32_t grid,
                             dsq_cuda_stack** out) {
    return stack_create_impl(layers, n, deps, xs, ys, y_dtype, reduce, tp, grid, out);
}

int dsq_cuda_stack_create_batch(dsq_cuda_layer* const* layers, uint32_t n, const int32_t* deps,
                                const void* const* xs, void* const* ys, int y_dtype,
                                uint32_t batch, uint32_t x_bstride, uint32_t y_bstride,
                                dsq_cuda_stack** out) {
    return stack_create_impl(layers, n, deps, xs, ys, y_dtype, nullptr, nullptr, 0, out, batch,
                             x_bstride, y_bstride);
}

// ---- tensor-parallel context: this rank's receive buffer + flags, peers mapped
int dsq_cuda_tp_create(int device, uint32_t world, uint32_t rank, uint32_t max_rows,
                       uint32_t max_grid, dsq_cuda_tp** out, void* ipc_handle) {
    if (!out || world < 1 || world > 8 || rank >= world || max_rows == 0 || max_grid == 0)
        return fail(DSQ_E_INVALID_ARGUMENT, "tp: world 1..8, rank < world, sizes > 0");
    *out = nullptr;
    CUDA_TRY(cudaSetDevice(device));
    auto* t = new dsq_cuda_tp;
    t->device = device;
    t->world = world;
    t->rank = rank;
    t->max_rows = (max_rows + 3) & ~3u;
    t->max_grid = max_grid;
    t->recv_bytes = size_t(2) * world * t->max_rows * 8;  // {value, tag} words
    const size_t bytes = t->recv_bytes + 16;                // + watchdog flag
    cudaError_t e = cudaMalloc(&t->buf, bytes);
    if (e == cudaSuccess) e = cudaMemset(t->buf, 0, bytes);
    if (e == cudaSuccess && ipc_handle) {
        cudaIpcMemHandle_t h;
        e = cudaIpcGetMemHandle(&h, t->buf);
        if (e == cudaSuccess) std::memcpy(ipc_handle, &h, sizeof(h));
    }
    if (e != cudaSuccess) {
        if (t->buf) cudaFree(t->buf);
        delete t;
        return cuda_fail(e, "tp buffer");
    }
    t->peer_base[rank] = t->buf;
    *out = t;
    return DSQ_OK;
}

int dsq_cuda_tp_connect(dsq_cuda_tp* t, const void* handles) {
    if (!t || !handles) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    CUDA_TRY(cudaSetDevice(t->device));
    for (uint32_t k = 0; k < t->world; ++k) {
        if (k == t->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t*>(handles) + k * sizeof(h), sizeof(h));
        void* p = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        t->peer_base[k] = p;
        t->peer_ipc[k] = true;
    }
    return DSQ_OK;
}

int dsq_cuda_tp_connect_local(dsq_cuda_tp* const* ctxs, uint32_t world) {
    if (!ctxs || world < 1 || world > 8) return fail(DSQ_E_INVALID_ARGUMENT, "bad contexts");
    for (uint32_t r = 0; r < world; ++r) {
        if (!ctxs[r] || ctxs[r]->world != world || ctxs[r]->rank != r)
            return fail(DSQ_E_INVALID_ARGUMENT, "tp: context %u has the wrong world/rank", r);
        for (uint32_t k = 0; k < world; ++k) ctxs[r]->peer_base[k] = ctxs[k]->buf;
    }
    return DSQ_OK;
}

int dsq_cuda_tp_error(const dsq_cuda_tp* t) {
    if (!t) return fail(DSQ_E_INVALID_ARGUMENT, "null tp");
    cudaSetDevice(t->device);
    uint32_t v = 0;
    CUDA_TRY(cudaMemcpy(&v, static_cast<const uint8_t*>(t->buf) + t->recv_bytes, 4,
                        cudaMemcpyDeviceToHost));
    return v ? fail(DSQ_E_INTERNAL, "tp: a peer never arrived (watchdog fired)") : DSQ_OK;
}

int dsq_cuda_tp_destroy(dsq_cuda_tp* t) {
    if (!t) return DSQ_OK;
    cudaSetDevice(t->device);
    for (uint32_t k = 0; k < t->world; ++k)
        if (t->peer_ipc[k]) cudaIpcCloseMemHandle(t->peer_base[k]);
    if (t->buf) cudaFree(t->buf);
    delete t;
    return DSQ_OK;
}

// debug: copy the stack timeline (grid * n * kTrSlots u64) to host; returns
// the number of u64 written (0 if tracing is off)
extern "C" uint64_t dsq_cuda_stack_trace(dsq_cuda_stack* S, unsigned long long* host,
                                         uint64_t cap) {
    if (!S || !S->trace) return 0;
    const uint64_t n = std::max<uint64_t>(uint64_t(S->sp.grid) * S->n * kTrSlots,
                                          uint64_t(S->sp.grid) * 24 * 5);
    if (cap < n) return 0;
    cudaSetDevice(S->device);
    cudaMemcpy(host, S->trace, n * 8, cudaMemcpyDeviceToHost);
    return n;
}

// one decode step from host memory: x_host -> x_dev, the stack, y_dev ->
// y_host, stream synchronised -- the host-buffer form of dsq_cuda_stack_run
int dsq_cuda_stack_run_host(dsq_cuda_stack* S, const void* x_host, void* x_dev, size_t x_bytes,
                            const void* y_dev, void* y_host, size_t y_bytes, void* stream) {
    if (!S) return fail(DSQ_E_INVALID_ARGUMENT, "null stack");
    if ((x_bytes && (!x_host || !x_dev)) || (y_bytes && (!y_dev || !y_host)))
        return fail(DSQ_E_INVALID_ARGUMENT, "stack_run_host: null buffer");
    cudaSetDevice(S->device);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (x_bytes) {
        // pinned (device-mapped) host x, 16-byte multiple: the GPU reads it
        // itself, overlapped with the stack kernel's prologue; else a memcpy
        cudaPointerAttributes at{};
        const bool mapped = cudaPointerGetAttributes(&at, x_host) == cudaSuccess &&
                            at.type == cudaMemoryTypeHost && at.devicePointer == x_host &&
                            !(reinterpret_cast<uintptr_t>(x_host) & 15u) &&
                            !(reinterpret_cast<uintptr_t>(x_dev) & 15u) && x_bytes % 16 == 0;
        cudaGetLastError();
        if (mapped && !S->seq)
            CUDA_TRY(launch_upload_x(x_host, x_dev, x_bytes, st));
        else
            CUDA_TRY(cudaMemcpyAsync(x_dev, x_host, x_bytes, cudaMemcpyHostToDevice, st));
    }
    const int rc = dsq_cuda_stack_run(S, stream);
    if (rc) return rc;
    if (y_bytes) CUDA_TRY(cudaMemcpyAsync(y_host, y_dev, y_bytes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return DSQ_OK;
}

int dsq_cuda_stack_run(dsq_cuda_stack* S, void* stream) {
    if (!S) return fail(DSQ_E_INVALID_ARGUMENT, "null stack");
    if (S->serve_dev) return fail(DSQ_E_INVALID_ARGUMENT, "served stack: use dsq_cuda_serve_*");
    cudaSetDevice(S->device);
    if (S->seq) {
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        auto enqueue = [&](cudaStream_t s) -> int {
            uint32_t launches = 0;
            for (const StackSeqStep& q : S->steps) {
                const int rc = gemv_impl(q.layer, DSQ_KERNEL_FUSED, q.x, DSQ_F16, q.y,
                                         int(S->y_dtype), S->batch, s, true, q.x_stride, q.y_stride);
                if (rc) return rc;
                launches += S->batch == 1 || batch_route(q.layer, S->batch) == BatchRoute::k7 ? 1u : 2u;
            }
            S->launches = launches;
            return DSQ_OK;
        };
        if (S->seq_graph) {
            CUDA_TRY(cudaGraphLaunch(S->seq_graph, st));
            return DSQ_OK;
        }
        // first run: eager (creates the layers' batched plans and scratch),
        // then capture the same launches on an internal stream while the GPU
        // executes them; later runs are one graph launch, so the host never
        // paces the ~2 launches per layer
        const int rc0 = enqueue(st);
        if (rc0 || S->seq_runs++ > 0) return rc0;
        if (!S->seq_capture)
            CUDA_TRY(cudaStreamCreateWithFlags(&S->seq_capture, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamBeginCapture(S->seq_capture, cudaStreamCaptureModeThreadLocal));
        const int rc = enqueue(S->seq_capture);
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(S->seq_capture, &g);
        if (rc) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) return cuda_fail(e, "sequential stack capture");
        const cudaError_t e2 = cudaGraphInstantiate(&S->seq_graph, g, 0);
        cudaGraphDestroy(g);
        if (e2 != cudaSuccess) {
            S->seq_graph = nullptr;
            return cuda_fail(e2, "sequential stack graph");
        }
        return DSQ_OK;
    }
    if (S->tp) {
        // every rank runs the same sequence of launches, so the reduce
        // ordinals (and the peers' flag targets) stay in step
        S->sp.tp_base = uint32_t(S->tp->base);
        S->tp->base += S->n_reduce;
    }
    CUDA_TRY(launch_stack(S->sp, static_cast<cudaStream_t>(stream), true));
    return DSQ_OK;
}

int dsq_cuda_stack_info(const dsq_cuda_stack* S, uint32_t* persistent, uint32_t* launches) {
    if (!S) return fail(DSQ_E_INVALID_ARGUMENT, "null stack");
    if (persistent) *persistent = S->seq ? 0u : 1u;
    if (launches) *launches = S->launches;
    return DSQ_OK;
}

// ---- serving loop: one resident launch, the host feeds each step's x ----
int dsq_cuda_stack_create_served(dsq_cuda_layer* const* layers, uint32_t n, const int32_t* deps,
                                 const void* const* xs, void* const* ys, int y_dtype,
                                 const uint32_t* gate, const uint32_t* notify,
                                 dsq_cuda_stack** out) {
    if (!gate || !notify) return fail(DSQ_E_INVALID_ARGUMENT, "served stack: null gate / notify");
    uint32_t steps = 0, x_cols = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (gate[i] && (!deps || deps[i] >= 0))
            return fail(DSQ_E_INVALID_ARGUMENT, "served stack: gate on chained layer %u", i);
        // every gated layer of step k sits after notify k-1 and before notify
        // k (so gates never decrease, whatever ungated layers lie between)
        if (gate[i] && gate[i] != steps + 1)
            return fail(DSQ_E_INVALID_ARGUMENT,
                        "served stack: layer %u gated on step %u lies after notify %u", i, gate[i],
                        steps);
        if (gate[i] && layers && layers[i]) {
            if (x_cols && layers[i]->cols != x_cols)
                return fail(DSQ_E_SHAPE_MISMATCH, "served stack: gated layers' cols differ");
            x_cols = layers[i]->cols;
        }
        if (notify[i]) {
            if (notify[i] != steps + 1)
                return fail(DSQ_E_INVALID_ARGUMENT, "served stack: notify values must run 1, 2, ..");
            ++steps;
        }
    }
    for (uint32_t i = 0; i < n; ++i)
        if (gate[i] > steps)
            return fail(DSQ_E_INVALID_ARGUMENT, "served stack: gate %u beyond the last step", i);
    if (steps == 0) return fail(DSQ_E_INVALID_ARGUMENT, "served stack: no notify layer");
    const void* gx = nullptr;
    for (uint32_t i = 0; i < n; ++i)
        if (gate[i]) {
            if (gx && xs && xs[i] != gx)
                return fail(DSQ_E_INVALID_ARGUMENT, "served stack: gated layers must share one x");
            gx = xs ? xs[i] : nullptr;
        }
    size_t y_cap = SIZE_MAX;
    for (uint32_t i = 0; i < n; ++i)
        if (notify[i] && layers && layers[i] && ys && ys[i]) {
            const size_t yb = size_t(layers[i]->rows) * (y_dtype == DSQ_F16 ? 2 : 4);
            y_cap = (reinterpret_cast<uintptr_t>(ys[i]) & 15u) ? 0 : std::min(y_cap, yb);
        }
    int rc = stack_create_impl(layers, n, deps, xs, ys, y_dtype, nullptr, nullptr, 0, out);
    if (rc) return rc;
    dsq_cuda_stack* S = *out;
    auto bail = [&](cudaError_t e, const char* what) {
        dsq_cuda_stack_destroy(S);
        *out = nullptr;
        return cuda_fail(e, what);
    };
    if (S->seq) {
        dsq_cuda_stack_destroy(S);
        *out = nullptr;
        return fail(DSQ_E_UNSUPPORTED, "served stack: needs the persistent form");
    }
    // device: [gate n][notify n][flag][err]
    cudaError_t e = cudaMalloc(&S->serve_dev, (size_t(2) * n + 2) * 4);
    if (e != cudaSuccess) return bail(e, "served stack buffers");
    std::vector<uint32_t> h(size_t(2) * n + 2, 0);
    std::copy(gate, gate + n, h.begin());
    std::copy(notify, notify + n, h.begin() + n);
    if ((e = cudaMemcpy(S->serve_dev, h.data(), h.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
        return bail(e, "served stack upload");
    // pinned host: [0] host_done, [1] doorbell
    if ((e = cudaHostAlloc(reinterpret_cast<void**>(&S->serve_pin), 64,
                           cudaHostAllocMapped | cudaHostAllocPortable)) != cudaSuccess)
        return bail(e, "served stack pinned words");
    S->serve_pin[0] = S->serve_pin[1] = 0;
    uint32_t* pin_map = nullptr;
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&pin_map), S->serve_pin, 0)) !=
        cudaSuccess)
        return bail(e, "served stack host mapping");
    S->serve_steps = steps;
    S->serve_x_cols = x_cols;
    S->serve_y_cap = y_cap == SIZE_MAX ? 0 : y_cap;
    S->serve_x_ptr = gx;
    S->sp.serve_gate = S->serve_dev;
    S->sp.serve_notify = S->serve_dev + n;
    S->sp.serve_flag = S->serve_dev + 2 * n;
    S->sp.serve_err = S->serve_dev + 2 * n + 1;
    S->sp.host_done = pin_map;
    S->sp.doorbell = pin_map + 1;
    return DSQ_OK;
}

int dsq_cuda_serve_begin(dsq_cuda_stack* S, void* x_dev, size_t x_bytes, void* y_host,
                         size_t y_bytes, void* stream) {
    if (!S || !S->serve_dev) return fail(DSQ_E_INVALID_ARGUMENT, "serve: not a served stack");
    if (S->serving) return fail(DSQ_E_INVALID_ARGUMENT, "serve: already running");
    if (!x_dev || !x_bytes || x_bytes % 16 || (reinterpret_cast<uintptr_t>(x_dev) & 15u))
        return fail(DSQ_E_INVALID_ARGUMENT, "serve: x_dev / x_bytes must be 16-byte aligned, > 0");
    if (S->serve_x_ptr && x_dev != S->serve_x_ptr)
        return fail(DSQ_E_INVALID_ARGUMENT, "serve: x_dev is not the gated layers' x buffer");
    // CTA 0 writes exactly x_bytes into the gated layers' x every step
    if (S->serve_x_cols &&
        (x_bytes < size_t(S->serve_x_cols) * 2 || x_bytes > (size_t(S->serve_x_cols) * 2 + 15) / 16 * 16))
        return fail(DSQ_E_SHAPE_MISMATCH, "serve: x_bytes %zu does not match the gated layers' %u "
                    "fp16 columns", x_bytes, S->serve_x_cols);
    if (y_bytes % 16 || (y_bytes && (!y_host || (reinterpret_cast<uintptr_t>(y_host) & 15u))))
        return fail(DSQ_E_INVALID_ARGUMENT, "serve: y_host / y_bytes must be 16-byte aligned");
    cudaSetDevice(S->device);
    S->sp.serve_y_ll = nullptr;
    S->sp.serve_y_words = 0;
    S->serve_y_host = nullptr;
    if (y_bytes) {
        if (y_bytes > S->serve_y_cap)
            return fail(DSQ_E_INVALID_ARGUMENT,
                        "serve: y_bytes > a notify layer's output (or its y is not 16-byte aligned)");
        // the kernel's tagged output words (4 payload bytes each), cleared so
        // no tag of an earlier session matches
        const size_t ll_bytes = y_bytes * 2;
        if (S->serve_ll_cap < ll_bytes) {
            if (S->serve_ll_pin) cudaFreeHost(S->serve_ll_pin);
            S->serve_ll_pin = nullptr;
            S->serve_ll_cap = 0;
            CUDA_TRY(cudaHostAlloc(&S->serve_ll_pin, ll_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
            S->serve_ll_cap = ll_bytes;
        }
        std::memset(S->serve_ll_pin, 0, ll_bytes);
        void* ll_map = nullptr;
        CUDA_TRY(cudaHostGetDevicePointer(&ll_map, S->serve_ll_pin, 0));
        S->sp.serve_y_ll = static_cast<unsigned long long*>(ll_map);
        S->sp.serve_y_words = uint32_t(y_bytes / 4);
        S->serve_y_host = static_cast<uint32_t*>(y_host);
    }
    if (S->serve_x_cap < x_bytes) {
        if (S->serve_x_pin) cudaFreeHost(S->serve_x_pin);
        S->serve_x_pin = nullptr;
        S->serve_x_cap = 0;
        CUDA_TRY(cudaHostAlloc(&S->serve_x_pin, x_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
        S->serve_x_cap = x_bytes;
    }
    void* x_map = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(&x_map, S->serve_x_pin, 0));
    S->sp.serve_x_src = static_cast<const uint4*>(x_map);
    S->sp.serve_x_dst = static_cast<uint4*>(x_dev);
    S->sp.serve_x_bytes = uint32_t(x_bytes);
    S->serve_x_bytes = x_bytes;
    const uint32_t zero[2] = {0, 0};
    CUDA_TRY(cudaMemcpy(S->serve_dev + 2 * S->n, zero, 8, cudaMemcpyHostToDevice));  // flag, err
    reinterpret_cast<volatile uint32_t*>(S->serve_pin)[0] = 0;  // host_done
    reinterpret_cast<volatile uint32_t*>(S->serve_pin)[1] = 0;  // doorbell
    S->serve_k = 0;
    S->serve_stream = static_cast<cudaStream_t>(stream);
    CUDA_TRY(launch_stack(S->sp, S->serve_stream, false));
    S->serving = true;
    return DSQ_OK;
}

int dsq_cuda_serve_step(dsq_cuda_stack* S, const void* x_host) {
    if (!S || !S->serving) return fail(DSQ_E_INVALID_ARGUMENT, "serve: not running");
    if (S->serve_k >= S->serve_steps) return fail(DSQ_E_INVALID_ARGUMENT, "serve: no steps left");
    if (!x_host) return fail(DSQ_E_INVALID_ARGUMENT, "serve: null x");
    const uint32_t k = ++S->serve_k;
    // step k-1 is complete, so the kernel has copied its x out of the staging
    // buffer: refill it, then ring (x86 stores are seen in order over PCIe)
    std::memcpy(S->serve_x_pin, x_host, S->serve_x_bytes);
    std::atomic_thread_fence(std::memory_order_seq_cst);
    reinterpret_cast<volatile uint32_t*>(S->serve_pin)[1] = k;
    const auto t0 = std::chrono::steady_clock::now();
    uint32_t spins = 0;
    auto late = [&]() {
        return (++spins & 1023u) == 0 &&
               std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10);
    };
    if (S->serve_y_host) {
        // the step's output words, tag k each (written by the finishing warps
        // of the notify layer, no fence): spin per word, keep the payload
        const volatile unsigned long long* ll =
            static_cast<const volatile unsigned long long*>(S->serve_ll_pin);
        const uint32_t nw = S->sp.serve_y_words;
        for (uint32_t w = 0; w < nw; ++w) {
            unsigned long long v;
            while (uint32_t((v = ll[w]) >> 32) != k)
                if (late()) return fail(DSQ_E_INTERNAL, "serve: step %u did not complete in 10 s", k);
            S->serve_y_host[w] = uint32_t(v);
        }
        return DSQ_OK;
    }
    const volatile uint32_t* done = S->serve_pin;
    while (*done < k)
        if (late()) return fail(DSQ_E_INTERNAL, "serve: step %u did not complete in 10 s", k);
    std::atomic_thread_fence(std::memory_order_acquire);
    return DSQ_OK;
}

int dsq_cuda_serve_end(dsq_cuda_stack* S) {
    if (!S || !S->serving) return fail(DSQ_E_INVALID_ARGUMENT, "serve: not running");
    cudaSetDevice(S->device);
    if (S->serve_k < S->serve_steps)  // release the steps not fed (stale x)
        reinterpret_cast<volatile uint32_t*>(S->serve_pin)[1] = 0xffffffffu;
    S->serving = false;
    CUDA_TRY(cudaStreamSynchronize(S->serve_stream));
    uint32_t err = 0;
    CUDA_TRY(cudaMemcpy(&err, S->serve_dev + 2 * S->n + 1, 4, cudaMemcpyDeviceToHost));
    return err ? fail(DSQ_E_INTERNAL, "serve: kernel reported an error") : DSQ_OK;
}

int dsq_cuda_stack_destroy(dsq_cuda_stack* S) {
    if (!S) return DSQ_OK;
    cudaSetDevice(S->device);
    if (S->serving) {
        dsq_cuda_serve_end(S);
    }
    if (S->serve_x_pin) cudaFreeHost(S->serve_x_pin);
    if (S->serve_ll_pin) cudaFreeHost(S->serve_ll_pin);
    if (S->serve_pin) cudaFreeHost(S->serve_pin);
    if (S->serve_dev) cudaFree(S->serve_dev);
    if (S->arena) cudaFree(S->arena);
    if (S->trace) cudaFree(S->trace);
    if (S->seq_graph) cudaGraphExecDestroy(S->seq_graph);
    if (S->seq_capture) cudaStreamDestroy(S->seq_capture);
    delete S;
    return DSQ_OK;
}

int dsq_cuda_gemv_many(dsq_cuda_layer* const* layers, uint32_t n, int kernel,
                       const void* const* xs, int x_dtype, void* const* ys, int y_dtype,
                       void* stream) {
    if (!layers || !xs || !ys) return fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    for (uint32_t i = 0; i < n; ++i) {
        int rc = gemv_impl(layers[i], kernel, xs[i], x_dtype, ys[i], y_dtype, 1,
                           static_cast<cudaStream_t>(stream), true);
        if (rc) return rc;
    }
    return DSQ_OK;
}

}  // extern "C"
