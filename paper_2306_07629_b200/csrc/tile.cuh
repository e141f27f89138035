// tile.cuh -- the decode micro-kernel of the tile-record layout (stack.hpp):
// PRMT byte-plane LUT lookups build fp16 A fragments, mma.sync.m16n8k16
// accumulates the exact fp16 x fp16 products in fp32.
//
// Why tensor cores at batch 1: the path is issue-bound, not FLOP-bound.  With
// FHFMA the decode costs ~2.3 instructions per weight; moving the multiply-
// accumulate into HMMA leaves ~1.2 ALU instructions per weight (1 PRMT + the
// selector preparation) and 1/256 HMMA, which is what lets one SM keep up with
// its share of HBM (tools/microbench/hmma_mb.cu: 38 vs 28 weights/clk/SM).
//
// Block-diagonal fragment map (one warp, one 4-row tile, one 256-column span).
// The span's columns form 16 PIECES of 16: piece p = columns 8p + [0,8) and
// 128 + 8p + [0,8) (so the x of pieces 0..7 is two contiguous 128-byte runs).
//   lane = 4g + t, g = 4h + i  ->  tile row i, pieces pA = 4h + t, pB = 8 + 4h + t
//   the lane's 32 indices: idx[q] = piece pA position q, idx[16+q] = pB pos. q
//   HMMA j (j = 0..3): a0/a2 = row i, pA positions 4j..4j+3      (A row g)
//                      a1/a3 = row i, pB positions 4j..4j+3      (A row g+8)
//   so A row m = 4*blk + i covers tile row i on piece set blk (blk = m/4),
//   B column n = blk carries x of piece 4n + t (lanes with g&3 == n load it:
//   conflict-free LDS.128s, 8 lanes read 128 contiguous bytes),
//   and y_i = D[i][0] + D[4+i][1] + D[8+i][2] + D[12+i][3].
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

namespace sqz {

__device__ __forceinline__ void hmma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// bits 16..31 -> bits 0..15 on the FMA pipe (the ALU pipe is the bottleneck):
// an fp16 multiply by 1.0 of the upper half.  Selector halves have bit 3 of
// every nibble clear, so they are finite fp16 values and the copy is exact.
__device__ __forceinline__ uint32_t hi16(uint32_t a) {
    uint32_t r;
    asm("{.reg .b16 l, h, o, one;\n"
        " mov.b16 one, 0x3C00;\n"
        " mov.b32 {l, h}, %1;\n"
        " mul.rn.f16 o, h, one;\n"
        " mov.b32 %0, {o, o};}"
        : "=r"(r)
        : "r"(a));
    return r;
}

// quad lookup: 4 indices in the low 4 nibbles of s -> two fp16x2 words
__device__ __forceinline__ void quad8(uint32_t s, const Planes8& P, uint32_t& p01, uint32_t& p23) {
    const uint32_t lo = prmt(P.l0, P.l1, s);
    const uint32_t hi = prmt(P.h0, P.h1, s);
    p01 = prmt(lo, hi, 0x5140);
    p23 = prmt(lo, hi, 0x7362);
}

// 16-entry quad lookup: pk picks entries 8..15 (nibble 4+n) or 0..7 (n)
__device__ __forceinline__ void quad16(uint32_t s, uint32_t pk, const Planes16& P, uint32_t& p01,
                                       uint32_t& p23) {
    const uint32_t loA = prmt(P.a.l0, P.a.l1, s), loB = prmt(P.b.l0, P.b.l1, s);
    const uint32_t hiA = prmt(P.a.h0, P.a.h1, s), hiB = prmt(P.b.h0, P.b.h1, s);
    const uint32_t lo = prmt(loA, loB, pk), hi = prmt(hiA, hiB, pk);
    p01 = prmt(lo, hi, 0x5140);
    p23 = prmt(lo, hi, 0x7362);
}

// Shift / subtract constants in registers the compiler cannot see through
// (kernel parameters set by the host, see kShiftK), so mul.hi / mad.lo stay
// IMAD.HI / IMAD on the FMA pipe instead of being strength-reduced back to
// ALU shifts and ANDs: k29/k30/k31 = 2^29/2^30/2^31 (mul.hi by 2^(32-s) is a
// right shift by s), kneg = 0xffffffff (w + m * kneg = w - m).
struct ShiftK {
    uint32_t k29, k30, k31, kneg;
};
#define SQZ_SHIFTK_INIT {1u << 29, 1u << 30, 1u << 31, 0xffffffffu}

// The decode of one lane's share of one (tile, span) unit, written once:
// every product variant (and the fragment dump of the parity tests,
// stack.cu dump_frags) runs these and hands the A fragments of HMMA j
// (j = 0..3) to its sink.
//
// 3-bit, words w0..w2 ("nibble + spare", layout.hpp).  ALU pipe: the three
// selector masks m_k = w_k & 0x77777777, the spare-index gather
// t = (w0>>3 & 0x1..) | (w1>>2 & 0x2..) | (w2>>1 & 0x4..) and the 32 PRMTs;
// FMA pipe: the hi16 selector halves (HMUL2).  (DSQ_IMAD_GATHER moves the
// gather to the FMA pipe -- e_k = w_k - m_k by IMAD, three chained IMAD.HI --
// which cuts 6 ALU instructions per unit but measured 6% slower on B200: the
// unit loop is bound by issue latency, not by the ALU pipe.)
template <typename Sink>
__device__ __forceinline__ void span3_frags(uint32_t w0, uint32_t w1, uint32_t w2,
                                            const Planes8& P, Sink&& sink, const ShiftK& K) {
    const uint32_t m0 = w0 & 0x77777777u, m1 = w1 & 0x77777777u, m2 = w2 & 0x77777777u;
#ifndef DSQ_IMAD_GATHER  // the gather on the ALU pipe (3 SHF + 3 LOP3); see below
    (void)K;
    const uint32_t t =
        ((w0 >> 3) & 0x11111111u) | ((w1 >> 2) & 0x22222222u) | ((w2 >> 1) & 0x44444444u);
#else  // dev variant: on the FMA pipe -- measured 6% slower (longer dependency chain)
    uint32_t e0, e1, e2, a, b, t;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(e0) : "r"(m0), "r"(K.kneg), "r"(w0));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(e1) : "r"(m1), "r"(K.kneg), "r"(w1));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(e2) : "r"(m2), "r"(K.kneg), "r"(w2));
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(a) : "r"(e2), "r"(K.k31));
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(b) : "r"(e1), "r"(K.k30), "r"(a));
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(e0), "r"(K.k29), "r"(b));
#endif
    const uint32_t sA[4] = {m0, hi16(m0), m1, hi16(m1)};
    const uint32_t sB[4] = {m2, hi16(m2), t, hi16(t)};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint32_t a0, a1, a2, a3;
        quad8(sA[j], P, a0, a2);
        quad8(sB[j], P, a1, a3);
        sink(j, a0, a1, a2, a3);
    }
}

// 4-bit: words w[0..3] (nibble n of w[k] = index 8k+n)
template <typename Sink>
__device__ __forceinline__ void span4_frags(const uint4& w, const Planes16& P, Sink&& sink) {
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    uint32_t sl[4], pk[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        sl[q] = ws[q] & 0x77777777u;
        pk[q] = ((ws[q] >> 1) & 0x44444444u) | 0x32103210u;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int wa = j >> 1, wb = 2 + (j >> 1);
        const uint32_t sa = (j & 1) ? hi16(sl[wa]) : sl[wa];
        const uint32_t pa = (j & 1) ? hi16(pk[wa]) : pk[wa];
        const uint32_t sb = (j & 1) ? hi16(sl[wb]) : sl[wb];
        const uint32_t pb = (j & 1) ? hi16(pk[wb]) : pk[wb];
        uint32_t a0, a1, a2, a3;
        quad16(sa, pa, P, a0, a2);
        quad16(sb, pb, P, a1, a3);
        sink(j, a0, a1, a2, a3);
    }
}

// 3-bit unit -> 4 HMMAs into two accumulator sets (breaks the HMMA chain)
__device__ __forceinline__ void span3_mma(uint32_t w0, uint32_t w1, uint32_t w2, const Planes8& P,
                                          const uint4& xa, const uint4& xb, float (&d0)[4],
                                          float (&d1)[4], const ShiftK& K) {
    const uint32_t xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
    span3_frags(
        w0, w1, w2, P,
        [&](int j, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
            if (j & 1)
                hmma16816(d1, a0, a1, a2, a3, xs[2 * j], xs[2 * j + 1]);
            else
                hmma16816(d0, a0, a1, a2, a3, xs[2 * j], xs[2 * j + 1]);
        },
        K);
}

// the same for one unit into a single accumulator set; two independent units
// interleaved (span pairs) give the scheduler twice the independent work
__device__ __forceinline__ void span3_mma_one(uint32_t w0, uint32_t w1, uint32_t w2,
                                              const Planes8& P, const uint4& xa, const uint4& xb,
                                              float (&d)[4], const ShiftK& K) {
    const uint32_t xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
    span3_frags(
        w0, w1, w2, P,
        [&](int j, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
            hmma16816(d, a0, a1, a2, a3, xs[2 * j], xs[2 * j + 1]);
        },
        K);
}

// batch 3..8: the same A fragments against NX more x sets (vector pairs
// 2/3, 4/5, 6/7) into NX more accumulator pairs -- decode paid once
template <int NX>
__device__ __forceinline__ void span3_mma_xn(uint32_t w0, uint32_t w1, uint32_t w2,
                                             const Planes8& P, const uint4& xa, const uint4& xb,
                                             const uint4 (&ya)[NX], const uint4 (&yb)[NX],
                                             float (&d0)[4], float (&d1)[4],
                                             float (&e)[NX][2][4], const ShiftK& K) {
    const uint32_t xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
    span3_frags(
        w0, w1, w2, P,
        [&](int j, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
            hmma16816((j & 1) ? d1 : d0, a0, a1, a2, a3, xs[2 * j], xs[2 * j + 1]);
#pragma unroll
            for (int q = 0; q < NX; ++q) {
                const uint4& A = (j < 2) ? ya[q] : yb[q];
                const uint32_t y0 = (j & 1) ? A.z : A.x, y1 = (j & 1) ? A.w : A.y;
                hmma16816(e[q][j & 1], a0, a1, a2, a3, y0, y1);
            }
        },
        K);
}

__device__ __forceinline__ void span4_mma(const uint4& w, const Planes16& P, const uint4& xa,
                                          const uint4& xb, float (&d0)[4], float (&d1)[4]) {
    const uint32_t xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
    span4_frags(w, P, [&](int j, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
        if (j & 1)
            hmma16816(d1, a0, a1, a2, a3, xs[2 * j], xs[2 * j + 1]);
        else
            hmma16816(d0, a0, a1, a2, a3, xs[2 * j], xs[2 * j + 1]);
    });
}

template <int NX>
__device__ __forceinline__ void span4_mma_xn(const uint4& w, const Planes16& P, const uint4& xa,
                                             const uint4& xb, const uint4 (&ya)[NX],
                                             const uint4 (&yb)[NX], float (&d0)[4],
                                             float (&d1)[4], float (&e)[NX][2][4]) {
    const uint32_t xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
    span4_frags(w, P, [&](int j, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
        hmma16816((j & 1) ? d1 : d0, a0, a1, a2, a3, xs[2 * j], xs[2 * j + 1]);
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const uint4& A = (j < 2) ? ya[q] : yb[q];
            const uint32_t y0 = (j & 1) ? A.z : A.x, y1 = (j & 1) ? A.w : A.y;
            hmma16816(e[q][j & 1], a0, a1, a2, a3, y0, y1);
        }
    });
}

// position q (0..31) of the lane's 32 indices held by A register r (a0..a3)
// half h of HMMA j (the block-diagonal map above): a0/a2 = piece pA,
// a1/a3 = piece pB, a2/a3 = positions 4j+2, 4j+3
__host__ __device__ inline uint32_t frag_pos(int j, int r, int h) {
    return (r & 1 ? 16u : 0u) + 4u * j + (r & 2 ? 2u : 0u) + uint32_t(h);
}

// D fragments -> the 4 row sums of the tile in lanes 0, 4, 8, 12 (fixed order)
__device__ __forceinline__ float tile_rows_reduce(const float (&d0)[4], const float (&d1)[4],
                                                  uint32_t lane) {
    const uint32_t g = lane >> 2, t = lane & 3;
    const float c0 = d0[0] + d1[0], c1 = d0[1] + d1[1], c2 = d0[2] + d1[2], c3 = d0[3] + d1[3];
    float v = t == 0 ? (g < 4 ? c0 : c1) : (t == 1 ? (g < 4 ? c2 : c3) : 0.f);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    return v;
}

// the same for two batch vectors (B columns 0-3 = vector 0, 4-7 = vector 1):
// row i of vector 0 lands in lane 4i, of vector 1 in lane 4i + 2
__device__ __forceinline__ float tile_rows_reduce2(const float (&d0)[4], const float (&d1)[4],
                                                   uint32_t lane) {
    const uint32_t g = lane >> 2, t = lane & 3;
    const float c0 = d0[0] + d1[0], c1 = d0[1] + d1[1], c2 = d0[2] + d1[2], c3 = d0[3] + d1[3];
    float v = (t & 1) == 0 ? (g < 4 ? c0 : c1) : (g < 4 ? c2 : c3);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    return v;
}

// x halves a lane feeds into B: 8 halves at this offset within the span and
// 8 more at +128 (piece 4n + t, n = B column)
__device__ __forceinline__ uint32_t tile_x_offset(uint32_t lane) {
    const uint32_t n = (lane >> 2) & 3u, t = lane & 3u;
    return 8u * (4u * n + t);
}

}  // namespace sqz
