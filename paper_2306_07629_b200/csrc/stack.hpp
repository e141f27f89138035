// stack.hpp -- persistent multi-layer decode kernel ("stack"), shared by the
// host (api.cpp) and the device (stack.cu).
//
// Row-record layout (bits 3/4, the path the stack kernel serves): every row r
// of a layer is one contiguous record of RW 32-bit words
//     [ LUT byte planes: 4 words (3-bit) | 8 words (4-bit) ]
//     [ index words, group-major: word k of group g at LW + g*bits + k ]
// where NG = ceil(cols/32) groups of 32 columns, NGP = NG rounded up to a
// multiple of 4 (16-byte records), and a group's `bits` words carry its 32
// indices in the encoding of layout.hpp.  Lanes of a warp take consecutive
// groups; with a 3-word (3-bit) stride the 32 lanes hit 32 distinct banks
// (gcd(3,32) = 1) and with a 4-word stride (4-bit) one LDS.128 per lane is a
// conflict-free 4-wavefront load, each lane using immediate offsets only.
// The LUT is stored as PRMT byte planes (lo bytes of e0..e3, e4..e7, hi bytes
// of e0..e3, e4..e7 -- same 16 bytes as the fp16 LUT, pre-transposed) so no
// per-row conversion is needed.  A CTA's share of a layer is a contiguous row
// range, i.e. a contiguous byte range -> plain TMA bulk copies.
#pragma once

#include <cstdint>

namespace sqz {

constexpr int kStackConsumersDefault = 16;  // decode warps per CTA (8/16/24; DSQ_STACK_CONSUMERS)
constexpr uint32_t kNoDep = 0xffffffffu;
constexpr uint32_t kInlineLayers = 8;  // layer descs carried in the launch params

struct StackLayerDesc {
    const uint32_t* rec;      // row records [rows][rw]
    const uint32_t* row_ptr;  // CSR row pointers [rows+1]
    const uint32_t* csr;      // CSR entries: col | fp16(delta) << 16
    const uint16_t* x;        // fp16 input [cols]
    void* y;                  // output [rows], fp16 or fp32
    uint32_t rows, cols, ng, ngp;
    uint32_t rw;              // words per row record
    uint32_t chunk_rows;      // max rows per ring slot (CTA shares split evenly)
    uint32_t dep;             // layer whose output is x (kNoDep: external input)
    uint32_t y_f16;
    uint32_t nslices;         // ceil(ng / 32)
    // host-precomputed row split over the grid (no device division):
    // CTA c owns rows [c*rq + min(c, rr), ...) -- rq or rq+1 rows -- cut into
    // fixed chunks of chunk_rows (nch_lo / nch_hi chunks for rq / rq+1 rows)
    uint32_t rq, rr, nch_lo, nch_hi;
};

struct StackParams {
    const StackLayerDesc* layers;    // device table, used when n_layers > kInlineLayers
    StackLayerDesc inl[kInlineLayers];
    uint32_t n_layers;
    uint32_t bits;
    uint32_t* counters;       // [n_layers + 1] completion counts (self-resetting)
    float* gseg;              // global spill for CSR round results [G][gseg_rounds][32]
    uint32_t gseg_rounds;
    uint32_t grid;            // CTAs (== SMs, all co-resident)
    uint32_t consumers;       // decode warps per CTA (+ producer, loader, finisher warps)
    // dynamic shared memory carve-up (byte offsets)
    uint32_t off_ring, slot_bytes, n_slots;
    uint32_t off_x, x_bytes;         // two x buffers
    uint32_t off_rp, rp_words;       // two row_ptr slices
    uint32_t off_csr, csr_cap;       // two CSR entry buffers (entries)
    uint32_t off_part, part_stride, part_rows;  // two per-(row, slice) partial buffers
    uint32_t off_seg, seg_rounds;    // CSR round scan results (rounds x 32 floats)
    uint32_t smem_bytes;
    // optional timeline (null = off): [grid][n_layers][kTraceSlots] globaltimer ns
    unsigned long long* trace;
};

// trace slots per (CTA, layer)
enum : uint32_t {
    kTrLoaderStart = 0,  // loader begins the layer (after its xempty wait)
    kTrCsrStaged,        // CSR slice staged
    kTrDepMet,           // dependency counter reached the grid size
    kTrXIssued,          // x TMA issued
    kTrConsStart,        // consumer warp 0 begins the layer
    kTrXReady,           // consumer warp 0 sees x
    kTrDenseDone,        // consumer warp 0 finished its dense pairs
    kTrCsrDone,          // consumer warp 0 passed the CSR rounds barrier
    kTrSignaled,         // completion counter bumped
    kTrProdFirst,        // producer issued the layer's first chunk
    kTrAllDense,         // finisher: all consumer warps done (pfull)
    kTrFinalDone,        // finisher: row totals stored (before the release)
    kTrSlots
};

}  // namespace sqz
