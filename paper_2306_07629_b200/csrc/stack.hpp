// stack.hpp -- persistent multi-layer decode kernel ("stack"), shared by the
// host (api.cpp) and the device (stack.cu).
//
// Tile layout (bits 3/4, the path the stack kernel serves).  Rows are grouped
// in TILES of 4 (rows padded to a multiple of 4 with all-zero LUTs); columns
// in SPANS of 256 (padded with index 0; x is zero-padded on chip).  A layer
// is two arrays:
//
//   lut [tiles][4 rows][LW words]   LUT byte planes of each row
//       LW = 4 (3-bit): lo bytes e0..e3 | lo e4..e7 | hi e0..e3 | hi e4..e7
//       LW = 8 (4-bit): the same for entries 0..7, then for 8..15
//   idx [tiles][NS spans][32 lanes x BITS words]   one UNIT = (tile, span)
//       lane = 16*h + 4*i + t  (i = row of the tile, h = 0/1, t = 0..3)
//       carries 32 indices of row i, columns 256*s + tile_col(h, t, q),
//       q = 0..31, in the "nibble + spare" encoding of layout.hpp; word order
//       3-bit: [k][lane] (three conflict-free LDS.32)
//       4-bit: [lane][k] (one conflict-free LDS.128)
//
// The lane -> (row, columns) map is the A-fragment map of a block-diagonal
// mma.sync.m16n8k16: A row m = 4*blk + i holds tile row i on piece set blk,
// B column n = blk holds x on those pieces, so one HMMA covers 4 rows x 64
// columns and D[4*blk + i][blk] are the 4 partial dot products (tile.cuh).
// Bytes: exactly rows*cols*bits/8 + 16*rows (3-bit) for aligned shapes, the
// reference's charged bytes (packfmt.cpp:98-121).  A CTA's share of a layer
// is a contiguous tile range, so its units are one contiguous byte range of
// idx (streamed in fixed-size chunks of whole units) and its LUT planes one
// contiguous range of lut -> plain TMA bulk copies.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define SQZ_HD __host__ __device__
#else
#define SQZ_HD
#endif

namespace sqz {

constexpr int kStackConsumersDefault = 16;  // decode warps per CTA (8/16; DSQ_STACK_CONSUMERS)
constexpr uint32_t kNoDep = 0xffffffffu;
constexpr uint32_t kInlineLayers = 8;  // layer descs carried in the launch params
constexpr uint32_t kTileRows = 4;
constexpr uint32_t kSpanCols = 256;
constexpr uint32_t kWarpSlotsDefault = 2;  // TMA ring slots per consumer warp (DSQ_STACK_SLOTS)
constexpr uint32_t kMaxWarpSlots = 6;      // mbarrier area: 16 x 6 + 30 barriers in 1 KB

// span column (0..255) of index position q (0..31) of lane (h, i, t): the
// lane covers pieces 4h+t (q < 16) and 8+4h+t (q >= 16); piece p is columns
// 8p + [0,8) then 128 + 8p + [0,8)  (tile.cuh)
SQZ_HD inline uint32_t tile_col(uint32_t h, uint32_t t, uint32_t q) {
    const uint32_t piece = (q < 16 ? 0u : 8u) + 4u * h + t, pos = q & 15u;
    return (pos < 8 ? 0u : 128u) + 8u * piece + (pos & 7u);
}

inline uint32_t tile_lut_words(uint32_t bits) { return bits == 3 ? 4u : 8u; }  // per row
inline uint32_t unit_words(uint32_t bits) { return bits * 32u; }

struct StackLayerDesc {
    const uint32_t* idx;        // index units [tiles][ns][bits*32]
    const uint32_t* lut;        // LUT planes [tiles][4][LW]
    const uint32_t* row_ptr;    // CSR row pointers [rows+1]
    const uint32_t* csr;        // CSR entries: col | fp16(delta) << 16
    const uint32_t* csr_rng;    // per CTA {row_ptr[r0], row_ptr[r1]} of its rows [grid][2]
    const uint32_t* csr_heads;  // bitmap: bit q set <=> entry q starts a row [nnz/32 + pad]
    const uint16_t* x;          // fp16 input [cols]
    void* y;                    // output [rows], fp16 or fp32
    uint32_t rows, cols;
    uint32_t tiles, ns;         // ceil(rows/4), ceil(cols/256)
    uint32_t dep;               // layer whose output is x (kNoDep: external input)
    uint32_t y_f16;
    uint32_t reduce_ord;        // TP: ordinal of this layer among the launch's partial-sum
                                // (row-parallel) layers, kNoDep if its y is final
    // host-precomputed tile split over the grid (no device division):
    // CTA c owns tiles [c*tq + min(c, tr), ...) -- tq or tq+1 tiles -- whose
    // units are streamed in chunks of cu units by the layer's first
    // nca = 1 << nca_shift consumer warps (the rest skip the layer: a layer
    // that gives a CTA few units runs on 8 of 16 warps, twice the units each)
    uint32_t tq, tr, cu, nca, nca_shift;
};

struct StackParams {
    const StackLayerDesc* layers;    // device table, used when n_layers > kInlineLayers
    StackLayerDesc inl[kInlineLayers];
    uint32_t n_layers;
    uint32_t bits;
    uint32_t* counters;       // [n_layers + 1] completion counts (self-resetting)
    float* gseg;              // global CSR scan results for CTAs beyond csr_cap [G][2][gseg_cap]
    uint32_t gseg_cap;
    uint32_t grid;            // CTAs (== SMs, all co-resident)
    uint32_t consumers;       // decode warps per CTA (+ producer, loader, finisher warps)
    uint32_t csr_warps;       // CSR / finishing warps (1..4)
    // dynamic shared memory carve-up (byte offsets)
    uint32_t off_desc;               // 8 x 128-byte layer descriptor cache
    uint32_t off_ring, slot_bytes, n_slots;
    uint32_t off_x, x_bytes;         // two x buffers
    uint32_t x_step;                 // bytes between them (0: one shared x buffer)
    uint32_t off_lut, lut_bytes;     // two LUT-plane buffers (the CTA's tiles)
    uint32_t off_rp, rp_words;       // two row_ptr slices
    uint32_t off_csr, csr_cap;       // two CSR entry buffers (entries)
    uint32_t off_hb, hb_words;       // two row-start bitmap buffers (words)
    uint32_t off_part, part_rows;    // two [consumers][part_rows] dense-partial buffers
    uint32_t off_seg, seg_cap;       // two CSR scan-result buffers (floats, position-indexed)
    uint32_t smem_bytes;
    // decode constants (tile.cuh ShiftK: 2^29, 2^30, 2^31, 0xffffffff), kept
    // opaque to the compiler so the spare-index gather stays on the FMA pipe
    uint32_t k29, k30, k31, kneg;
    // batch 2 (single-layer gemv): the two activation vectors share every
    // decoded A fragment -- vector b feeds the HMMA B columns 4b..4b+3, which
    // the block-diagonal map leaves free at batch 1.  x buffers, partial
    // tables and CSR scan buffers hold nbatch vectors each.
    uint32_t nbatch;                 // 1, 2 or 4 (vectors 2/3: a second HMMA per fragment)
    uint32_t nvec;                   // vectors actually supplied (<= nbatch; the rest are 0)
    uint32_t nbuf;                   // per-layer buffers (2; 1 for single-layer plans)
    uint32_t xvec;                   // halves between the vectors in an smem x buffer
    uint32_t x_bstride, y_bstride;   // elements between the vectors in global x / y
    // tensor parallelism (world > 1): the partial y of a reduce layer is
    // summed over the ranks' CTAs with the same index over peer memory.
    // recv = [2 parities][world][max_rows] {fp32 value, u32 tag} words per
    // rank; peer_recv are the (P2P-mapped) buffers of every rank, own rank
    // included; tp_flags[0] = watchdog error flag of this rank.
    uint32_t tp_world, tp_rank, tp_base, tp_max_rows;
    unsigned long long* tp_recv;
    uint32_t* tp_flags;
    unsigned long long* tp_peer_recv[8];
    // dev-only experiment switches (DSQ_STACK_DBG): bit 0 skips the decode math
    // (results are garbage; measures the streaming skeleton alone), bit 2
    // records the consumer cycle profile into `trace`
    uint32_t dbg;
    // optional timeline (null = off): [grid][n_layers][kTraceSlots] globaltimer ns
    unsigned long long* trace;
    // serving loop (dsq_cuda_serve_*; null = off).  A layer with serve_gate[l]
    // = k > 0 reads step k's input: CTA 0's loader waits for the host's
    // doorbell (*doorbell >= k, pinned host memory), copies the step's x from
    // the pinned staging buffer into serve_x_dst (the layer's x) over PCIe and
    // publishes *serve_flag = k; the other CTAs wait for the flag.  For a
    // layer with serve_notify[l] = k > 0 (fp16 y) every finishing warp
    // writes its rows straight into host memory as 64-bit words {two fp16
    // rows, tag k} (serve_y_ll, single-copy atomic: no fence, no gather --
    // the host polls the tags, NCCL's LL protocol idea); without an output
    // buffer CTA 0 waits for the layer's count, fences and stores k into
    // *host_done (pinned host memory).  No CUDA
    // call per step on the host.  The gate waits have no timeout (an idle
    // server may wait any time; a stale x is never computed on): only the
    // host's doorbell or serve_end's release (0xffffffff) ends them.
    const uint32_t* serve_gate;
    const uint32_t* serve_notify;
    const uint32_t* doorbell;     // device-mapped pinned host word
    const uint4* serve_x_src;     // device-mapped pinned staging, serve_x_bytes
    uint4* serve_x_dst;
    uint32_t serve_x_bytes;       // multiple of 16
    uint32_t* serve_flag;         // device word: the step whose x is in serve_x_dst
    unsigned long long* serve_y_ll;  // device-mapped pinned host: {rows 2j, 2j+1, tag} words
    uint32_t serve_y_words;       // rows / 2 of the notify layer's y sent (0: none)
    uint32_t* host_done;          // device-mapped pinned host word
    uint32_t* serve_err;
};

// trace slots per (CTA, layer)
enum : uint32_t {
    kTrLoaderStart = 0,  // loader begins the layer (after its xempty wait)
    kTrCsrStaged,        // CSR slice staged
    kTrDepMet,           // dependency counter reached the grid size
    kTrXIssued,          // x TMA issued
    kTrConsStart,        // consumer warp 0 begins the layer
    kTrXReady,           // consumer warp 0 sees x
    kTrDenseDone,        // consumer warp 0 finished its dense units
    kTrCsrDone,          // consumer warp 0 passed the CSR rounds barrier
    kTrSignaled,         // completion counter bumped
    kTrProdFirst,        // producer issued the layer's first chunk
    kTrAllDense,         // finisher: all consumer warps done (pfull)
    kTrFinalDone,        // finisher: row totals stored (before the release)
    kTrSlots
};

}  // namespace sqz
