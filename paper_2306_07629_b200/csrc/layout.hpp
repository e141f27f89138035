// layout.hpp -- device data layout of a quantized layer ("tiled" format) and
// the kernel parameter block.  Shared by the host packer/scheduler
// (packer.cpp, api.cpp) and the sm_100a kernels (kernels.cu).
//
// Reference layout (packfmt.hpp:16-33, packfmt.cpp:40-53): per row an
// LSB-first bitstream, index c at bits [c*bits, (c+1)*bits), rows padded to a
// byte.  That layout is neither coalesced across a warp nor aligned for
// vector loads, so the packer re-tiles it once at upload:
//
//   row block  = 32 consecutive rows (one per lane of a warp)
//   group      = 32 consecutive columns
//   unit u     = (row block rb, group g), u = rb * NG + g
//   unit bytes = 32 lanes x bits words  (32 indices x bits bits = bits words)
//   word order = [word k][lane]  -> a warp reads word k of a unit as one
//                128-byte coalesced, bank-conflict-free transaction
//
// Word encoding of the 32 indices idx[0..31] of one (row, group):
//   bits == 3 ("nibble + spare"):  w0 nibble n = idx[n]     | bit0(idx[24+n]) << 3
//                                  w1 nibble n = idx[8+n]   | bit1(idx[24+n]) << 3
//                                  w2 nibble n = idx[16+n]  | bit2(idx[24+n]) << 3
//     so w_k & 0x77777777 are ready-made PRMT byte selectors for 24 indices
//     and the remaining 8 are gathered from the bit-3 positions.
//   bits == 4: w_k nibble n = idx[8k + n]
//   other bits (1..8, generic path): a little-endian 32*bits-bit stream,
//     idx[j] at bits [j*bits, (j+1)*bits).
//
// Padding: rows are padded to a multiple of 32 (LUT zero), columns to a
// multiple of 32 (index 0; the kernels never read x beyond cols).
#pragma once

#include <cstdint>

namespace sqz {

constexpr uint32_t kRowBlock = 32;
constexpr uint32_t kGroupCols = 32;

// kernel geometry (fused LUT-GEMV)
constexpr int kWarpsPerCta = 8;
constexpr int kCtasPerSmDefault = 2;  // override with DSQ_CTAS_PER_SM (1..3)
constexpr int kMaxWorkers = 4096;      // warps in one balanced schedule
constexpr int kChunkUnits = 4;  // units per bulk copy
constexpr int kStages = 4;      // bulk-copy ring depth per warp

inline uint32_t ceil_div(uint64_t a, uint64_t b) { return uint32_t((a + b - 1) / b); }

// Parameter block of one layer's product, passed by value to the kernels.
struct LayerParams {
    const uint32_t* words;    // n_rb * NG * bits * 32 words (tiled indices)
    const uint16_t* lut;      // fp16 centroids [n_rb*32][2^bits]
    const uint32_t* row_ptr;  // CSR row pointers [rows+1]
    const uint32_t* csr;      // CSR entries: col | fp16(delta) << 16
    float* scratch;           // partial sums [2 * n_workers * 32] (first/last segment)
    uint32_t* counters;       // per row block arrival counters (self-resetting)
    uint32_t rows, cols, bits, n_rb, ng, n_workers, nnz;
};

// A grouped-LUT layer (groups_per_row > 1, kernels.cu grouped_gemv): the
// reference packed layout as is, LUTs per (row, column group).
struct GroupedParams {
    const uint8_t* payload;   // rows x stride bytes (reference layout)
    const uint16_t* lut;      // fp16 [rows][groups][K]
    const uint32_t* row_ptr;  // CSR row pointers [rows+1]
    const uint32_t* csr;      // col | fp16(delta) << 16
    uint32_t rows, cols, bits, groups, gcols, stride;
};

// The balanced schedule travels as a __grid_constant__ kernel parameter
// (constant bank, pushed with the launch): no dependent global load is needed
// before a warp knows its range.  Worker w owns units [u0[w], u0[w+1]).
struct WorkTable {
    uint32_t n;                     // workers
    uint32_t u0[kMaxWorkers + 1];   // strictly increasing, u0[0] = 0, u0[n] = units
};

}  // namespace sqz
