// bstream.cu -- K11: batched Dense-and-Sparse LUT-GEMM Y[b] = W X[b] for
// B = 5..16 activation vectors (BASELINE configs[4]) on per-warp TMA rings.
//
// Same HBM layout as the batch-1 kernel (stack.hpp: 4-row tiles, 256-column
// spans) read with a DENSE fragment map: a warp decodes a 16-row tile (4
// consecutive 4-row tiles) and every mma.sync.m16n8k16 uses all 16 A rows and
// all 8 B columns = 8 batch vectors, so one decoded weight feeds up to 16
// products for the tensor cost of batch 1 (B <= 8: 4 HMMA per 1024 weights,
// as the batch-1 block-diagonal map; B <= 16: 8).
//
//   thread (g, t): A rows g and g+8 = tile rows 16q + g and 16q + g + 8, i.e.
//   4-row tiles j0 = g / 4 and j0 + 2, tile row g % 4; it reads the two lanes
//   (h = 0/1, i = g % 4, t) of each of those tiles' units, 64 indices per row
//   per span = 16 quads; HMMA m takes quad m of both rows as its k-slots (2t,
//   2t+1, 2t+8, 2t+9) and x[vector g] at the quad's 4 columns as its B
//   fragment.  D[g][n] / D[g+8][n] are rows x vector n.
//
// Work split (host plan, bstream_plan below).  The columns are cut in PHASES
// of at most 8 (B > 8) or 16 spans, so one phase's x for all 8*NB vectors is
// 64 KB of shared memory; a CELL is (16-row tile q, span s) of a phase, ordered
// q-major.  Every CTA works in one phase on a contiguous cell range (CTAs per
// phase in proportion to the phase's cells), split again into 8 contiguous
// warp ranges.  Each warp streams its range through a private ring of 3 slots:
// a slot holds one CHUNK = up to cs consecutive spans of one 16-row tile, i.e.
// 4 bulk copies (one per 4-row tile, each a contiguous run of units) plus the
// tile's LUT planes, completed on one mbarrier.  The copies for the first
// three chunks are issued before the PDL wait (the weights are immutable), the
// phase's x is staged once per CTA after it.
//
// A warp flushes its accumulators when its range leaves a 16-row tile: one
// SEGMENT = the warp's partial products of that tile's 16 rows x 8*NB vectors
// (1 KB at NB = 2).  The host numbers the segments so that those of tile q,
// phase p are seg_base[p*T + q] .. seg_base[p*T + q + 1]; bstream_finish sums
// them in that fixed order, adds the CSR deltas, and writes y (deterministic,
// no atomics).  Segments cost ~(T*phases + warps) KB of L2-resident traffic,
// a few percent of the weight bytes at 7B shapes.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "bstream.hpp"
#include "ptx.cuh"
#include "stack.hpp"
#include "tile.cuh"

namespace sqz {

constexpr uint32_t kBsBarBytes = 512;  // mbarrier area at the start of shared memory
__host__ __device__ constexpr uint32_t bs_slots(uint32_t warps) { return warps == 16 ? 2u : 3u; }

struct BStreamParams {
    const uint32_t* idx;         // [tiles4][ns][UW]
    const uint32_t* lut;         // [tiles4][4][LW]
    const uint16_t* x;           // [B][x_stride] fp16, rows 16-byte aligned
    float* part;                 // [nseg][16][8*NB] segment partials
    uint16_t* xT;                // [ns*256][8*NB] x transposed for the CSR pass (or null)
    const uint4* wdesc;          // [grid*8] {cell_begin, cell_end, seg_first, bs_pack_w(phase, a, gp)}
    const uint32_t* seg_base;    // [phases*tiles16 + 1]
    uint32_t phases;
    uint32_t phase_span[kBsMaxPhases + 1];  // span boundaries of the phases
    uint32_t cta_pre[kBsMaxPhases + 1];     // CTAs of phase k: cta_pre[k] .. cta_pre[k+1]
    uint32_t cols, ns, tiles4, tiles16, B, x_stride;
    uint32_t xs_stride;    // halves per staged x row (max phase spans * 256 + 32)
    uint32_t cs;           // spans per chunk
    // slot layout (words): 4-row tiles 0, 1 at 0 and pw, the LUT planes of
    // all four at pw + cs*UW, tiles 2, 3 at pair and pair + pw.  pw = cs*UW +
    // 16 = 16 mod 32 keeps the two tiles one instruction reads on opposite
    // bank halves.
    uint32_t pw, pair, lut_off, slot_words;
};

// wdesc .w: phase (bits 0..7) | the CTA's index among the phase's CTAs
// (bits 8..19) | the phase's CTA count (bits 20..31) -- the CTAs of a phase
// write its transposed x between them
SQZ_HD inline uint32_t bs_pack_w(uint32_t phase, uint32_t a, uint32_t gp) {
    return phase | (a << 8) | (gp << 20);
}

// one lane's 32 indices of a unit -> 8 quads (selector words in the low 16
// bits; 4-bit: the pick words for the upper half table)
template <int BITS>
__device__ __forceinline__ void bs_quads(const uint32_t* w, uint32_t (&q)[8], uint32_t (&pk)[8]) {
    if constexpr (BITS == 3) {
        const uint32_t m0 = w[0] & 0x77777777u, m1 = w[1] & 0x77777777u, m2 = w[2] & 0x77777777u;
        const uint32_t t = ((w[0] >> 3) & 0x11111111u) | ((w[1] >> 2) & 0x22222222u) |
                           ((w[2] >> 1) & 0x44444444u);
        q[0] = m0; q[1] = hi16(m0); q[2] = m1; q[3] = hi16(m1);
        q[4] = m2; q[5] = hi16(m2); q[6] = t; q[7] = hi16(t);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t sl = w[k] & 0x77777777u;
            const uint32_t p = ((w[k] >> 1) & 0x44444444u) | 0x32103210u;
            q[2 * k] = sl;
            q[2 * k + 1] = hi16(sl);
            pk[2 * k] = p;
            pk[2 * k + 1] = hi16(p);
        }
    }
}

// one cell (16-row tile x one span) from the ring slot: u0 / u1 = the span's
// unit of the lane's 4-row tiles j0 / j0 + 2.  x B fragments: one LDS.128
// covers quads qi and qi + 1 (8 consecutive columns); with the staged rows
// 32 halves off a 64-half boundary the 8 lanes of each quarter-warp hit 32
// distinct banks.
template <int BITS, int NB>
__device__ __forceinline__ void bs_cell(const uint32_t* u0, const uint32_t* u1, uint32_t xcol,
                                        uint32_t i, uint32_t t, const Planes16& P0,
                                        const Planes16& P1, const uint16_t* xg0,
                                        const uint16_t* xg1, float (&d)[2][NB][4]) {
#pragma unroll
    for (uint32_t h = 0; h < 2; ++h) {
        const uint32_t L = 16 * h + 4 * i + t;
        uint32_t w0[BITS], w1[BITS];
        if constexpr (BITS == 3) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                w0[k] = u0[k * 32 + L];
                w1[k] = u1[k * 32 + L];
            }
        } else {
            const uint4 a = *reinterpret_cast<const uint4*>(u0 + L * 4);
            const uint4 b = *reinterpret_cast<const uint4*>(u1 + L * 4);
            w0[0] = a.x; w0[1] = a.y; w0[2] = a.z; w0[3] = a.w;
            w1[0] = b.x; w1[1] = b.y; w1[2] = b.z; w1[3] = b.w;
        }
        uint32_t q0[8], q1[8], k0[8], k1[8];
        bs_quads<BITS>(w0, q0, k0);
        bs_quads<BITS>(w1, q1, k1);
#pragma unroll
        for (uint32_t qp = 0; qp < 8; qp += 2) {
            const uint32_t col = xcol + tile_col(h, t, qp < 4 ? 4 * qp : 16 + 4 * (qp - 4));
            const uint4 xb = *reinterpret_cast<const uint4*>(xg0 + col);
            uint4 xc;
            if constexpr (NB == 2) xc = *reinterpret_cast<const uint4*>(xg1 + col);
#pragma unroll
            for (uint32_t e = 0; e < 2; ++e) {
                const uint32_t qi = qp + e;
                uint32_t a0, a1, a2, a3;
                if constexpr (BITS == 3) {
                    quad8(q0[qi], P0.a, a0, a2);
                    quad8(q1[qi], P1.a, a1, a3);
                } else {
                    quad16(q0[qi], k0[qi], P0, a0, a2);
                    quad16(q1[qi], k1[qi], P1, a1, a3);
                }
                hmma16816(d[h][0], a0, a1, a2, a3, e ? xb.z : xb.x, e ? xb.w : xb.y);
                if constexpr (NB == 2)
                    hmma16816(d[h][NB - 1], a0, a1, a2, a3, e ? xc.z : xc.x, e ? xc.w : xc.y);
            }
        }
    }
}

// NB = HMMA column groups (1: B <= 8, 2: B <= 16); W = decode warps per CTA
template <int BITS, int NB, int W>
__global__ void __launch_bounds__(W * 32, 1) bstream_gemv(const __grid_constant__ BStreamParams p) {
    constexpr int kBsWarps = W;
    constexpr int kBsSlots = int(bs_slots(W));
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t LW = BITS == 3 ? 4u : 8u;
    constexpr uint32_t UW = BITS * 32u;
    constexpr uint32_t NBV = 8u * NB;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + warp * kBsSlots;
    uint32_t* ring = reinterpret_cast<uint32_t*>(smem + kBsBarBytes) + warp * kBsSlots * p.slot_words;
    uint16_t* xs = reinterpret_cast<uint16_t*>(reinterpret_cast<uint32_t*>(smem + kBsBarBytes) +
                                               kBsWarps * kBsSlots * p.slot_words);
    // the warp's cell range from the launch parameters (no dependent load
    // before the first weight copies); its first segment id arrives by the
    // time the range first leaves a tile
    uint32_t phase, cta_a, cta_gp, cb, ce;
    bs_warp_range(p.phase_span, p.cta_pre, p.phases, p.tiles16, blockIdx.x, warp, W, &phase,
                  &cta_a, &cta_gp, &cb, &ce);
    const uint32_t sa = p.phase_span[phase], S = p.phase_span[phase + 1] - sa;
    const uint32_t seg_first = p.wdesc[blockIdx.x * kBsWarps + warp].z;
    // chunk at cell c: 16-row tile q = c / S, phase-local span c % S, up to cs
    // spans, not past the tile's last span or the warp's range
    auto issue = [&](uint32_t c, uint32_t slot, uint64_t pol) -> uint32_t {
        const uint32_t q = c / S, sl = c - q * S;
        const uint32_t n = min(min(p.cs, S - sl), ce - c);
        const uint32_t nt = min(4u, p.tiles4 - 4 * q);  // 4-row tiles that exist
        uint32_t* dst = ring + slot * p.slot_words;
        mbar_arrive_expect_tx(bar + slot, nt * (16u * LW + n * UW * 4u));
        bulk_g2s(dst + p.lut_off, p.lut + size_t(4 * q) * kTileRows * LW, nt * kTileRows * LW * 4u, bar + slot,
                 pol);
        for (uint32_t j = 0; j < nt; ++j)
            bulk_g2s(dst + (j & 1) * p.pw + (j >> 1) * p.pair,
                     p.idx + (size_t(4 * q + j) * p.ns + sa + sl) * UW, n * UW * 4u, bar + slot, pol);
        return c + n;
    };
    uint64_t* xbar = reinterpret_cast<uint64_t*>(smem) + kBsWarps * kBsSlots;
    uint32_t c_issue = cb;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kBsSlots; ++s) mbar_init(bar + s, 1);
        if (warp == 0) mbar_init(xbar, 1);
        fence_barrier_init();
        const uint64_t pol = policy_evict_first();
        for (int s = 0; s < kBsSlots && c_issue < ce; ++s) c_issue = issue(c_issue, s, pol);
    }
    // x, the segment buffer and xT may belong to the previous launch on this
    // stream (programmatic dependent launch): wait before touching them
    pdl_trigger();
    pdl_wait();
    {
        // the phase's x: the 16-byte-aligned body of each live vector row by
        // bulk copies on xbar (thread 0), the ragged tail and the rows of
        // vectors >= B by plain stores (disjoint bytes)
        const uint32_t c0 = sa * kSpanCols;
        const uint32_t ccount = min(p.cols, (sa + S) * kSpanCols) - min(p.cols, c0);
        const uint32_t body = ccount & ~7u;  // halves copied by TMA per row
        const uint32_t nlive = min(p.B, NBV);
        __syncthreads();  // xbar initialised
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(xbar, nlive * body * 2u);
            if (body)
                for (uint32_t b = 0; b < nlive; ++b)
                    bulk_g2s_plain(xs + b * p.xs_stride, p.x + size_t(b) * p.x_stride + c0, body * 2u,
                                   xbar);
        }
        const uint32_t rowh = S * kSpanCols;  // staged halves per row
        for (uint32_t b = warp; b < NBV; b += kBsWarps) {
            const uint32_t from = b < nlive ? body : 0u;
            for (uint32_t c = from + lane; c < rowh; c += 32)
                xs[b * p.xs_stride + c] = b < nlive && c < ccount ? p.x[size_t(b) * p.x_stride + c0 + c]
                                                                  : uint16_t(0);
        }
        __syncthreads();
        mbar_wait_spin(xbar, 0);
        if (p.xT) {
            // this CTA's share of the phase's transposed x: all vectors of a
            // column in one 16- / 32-byte run for the CSR gathers
            const uint32_t x0 = uint32_t(uint64_t(ccount) * cta_a / cta_gp);
            const uint32_t x1 = uint32_t(uint64_t(ccount) * (cta_a + 1) / cta_gp);
            for (uint32_t k = x0 * NB + threadIdx.x; k < x1 * NB; k += blockDim.x) {
                const uint32_t c = k / NB, j = k - c * NB;
                uint32_t h[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    h[e] = uint32_t(xs[(8 * j + 2 * e) * p.xs_stride + c]) |
                           (uint32_t(xs[(8 * j + 2 * e + 1) * p.xs_stride + c]) << 16);
                *reinterpret_cast<uint4*>(p.xT + size_t(c0 + c) * NBV + 8 * j) =
                    make_uint4(h[0], h[1], h[2], h[3]);
            }
        }
    }
    if (cb >= ce) return;
    const uint32_t g = lane >> 2, t = lane & 3, i = g & 3, j0 = g >> 2;  // rows g, g+8: tiles j0, j0+2
    const uint16_t* xg0 = xs + g * p.xs_stride;        // vector g
    const uint16_t* xg1 = xs + (8 + g) * p.xs_stride;  // vector 8 + g (NB == 2)
    // two accumulator sets (even / odd span of the unrolled pair), each with
    // one chain per h: 4 * NB independent HMMA chains
    float d[2][NB][4], e[2][NB][4];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int n = 0; n < NB; ++n)
#pragma unroll
            for (int r = 0; r < 4; ++r) d[c][n][r] = e[c][n][r] = 0.f;
    uint32_t seg = seg_first;
    uint32_t it = 0;
    for (uint32_t c = cb; c < ce;) {
        const uint32_t q = c / S, sl = c - q * S;
        const uint32_t n = min(min(p.cs, S - sl), ce - c);
        const uint32_t slot = it % kBsSlots;
        mbar_wait_spin(bar + slot, (it / kBsSlots) & 1u);
        const uint32_t* sw = ring + slot * p.slot_words;
        const bool v0 = 4 * q + j0 < p.tiles4, v1 = 4 * q + j0 + 2 < p.tiles4;
        Planes16 P0, P1;
        {
            const uint32_t* lt = sw + p.lut_off;
            const uint4 a0 = *reinterpret_cast<const uint4*>(lt + (j0 * 4 + i) * LW);
            const uint4 a1 = *reinterpret_cast<const uint4*>(lt + ((j0 + 2) * 4 + i) * LW);
            P0.a = v0 ? Planes8{a0.x, a0.y, a0.z, a0.w} : Planes8{0u, 0u, 0u, 0u};
            P1.a = v1 ? Planes8{a1.x, a1.y, a1.z, a1.w} : Planes8{0u, 0u, 0u, 0u};
            if constexpr (BITS == 4) {
                const uint4 b0 = *reinterpret_cast<const uint4*>(lt + (j0 * 4 + i) * LW + 4);
                const uint4 b1 = *reinterpret_cast<const uint4*>(lt + ((j0 + 2) * 4 + i) * LW + 4);
                P0.b = v0 ? Planes8{b0.x, b0.y, b0.z, b0.w} : Planes8{0u, 0u, 0u, 0u};
                P1.b = v1 ? Planes8{b1.x, b1.y, b1.z, b1.w} : Planes8{0u, 0u, 0u, 0u};
            }
        }
        const uint32_t* u0 = sw + j0 * p.pw;
        const uint32_t* u1 = u0 + p.pair;
        uint32_t u = 0;
        for (; u + 2 <= n; u += 2, u0 += 2 * UW, u1 += 2 * UW) {  // two spans: independent chains
            bs_cell<BITS, NB>(u0, u1, (sl + u) * kSpanCols, i, t, P0, P1, xg0, xg1, d);
            // 16 warps: one accumulator set (the registers of 512 threads)
            if constexpr (W == 16)
                bs_cell<BITS, NB>(u0 + UW, u1 + UW, (sl + u + 1) * kSpanCols, i, t, P0, P1, xg0, xg1, d);
            else
                bs_cell<BITS, NB>(u0 + UW, u1 + UW, (sl + u + 1) * kSpanCols, i, t, P0, P1, xg0, xg1, e);
        }
        if (u < n) bs_cell<BITS, NB>(u0, u1, (sl + u) * kSpanCols, i, t, P0, P1, xg0, xg1, d);
        // the slot's words are in registers or consumed: refill it
        __syncwarp();
        if (lane == 0 && c_issue < ce) c_issue = issue(c_issue, slot, policy_evict_first());
        ++it;
        c += n;
        if (c == ce || c - q * S == S) {
            // the range leaves tile q: one segment = D rows g / g+8, vectors 8n + 2t, +1
            float* out = p.part + size_t(seg) * 16 * NBV;
#pragma unroll
            for (int nn = 0; nn < NB; ++nn) {
                const uint32_t b0 = 8 * nn + 2 * t;
                *reinterpret_cast<float2*>(out + g * NBV + b0) =
                    make_float2((d[0][nn][0] + d[1][nn][0]) + (e[0][nn][0] + e[1][nn][0]),
                                (d[0][nn][1] + d[1][nn][1]) + (e[0][nn][1] + e[1][nn][1]));
                *reinterpret_cast<float2*>(out + (g + 8) * NBV + b0) =
                    make_float2((d[0][nn][2] + d[1][nn][2]) + (e[0][nn][2] + e[1][nn][2]),
                                (d[0][nn][3] + d[1][nn][3]) + (e[0][nn][3] + e[1][nn][3]));
#pragma unroll
                for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                    for (int r = 0; r < 4; ++r) d[cc][nn][r] = e[cc][nn][r] = 0.f;
            }
            // a later tile of this range starts with this warp: its first segment
            if (c < ce) seg = p.seg_base[phase * p.tiles16 + q + 1];
        }
    }
}

// y[b][r] = the row's segments + its CSR deltas.  One warp per row: lane =
// part * XB + b (XB = 8 * NB, P = 32 / XB parts).  Part k sums every P-th
// segment of each phase and every P-th CSR entry (entries in rounds of 32,
// one coalesced load per round); the parts are then added in a fixed shuffle
// order (deterministic).  All loads that do not
// depend on each other are issued together: the row pointers and the
// phases' segment bounds in one round trip, then the segments and the CSR
// entries, then the transposed x.
template <int XB>
__global__ void __launch_bounds__(256) bstream_finish(const float* __restrict__ part, const uint32_t* __restrict__ seg_base,
                               uint32_t phases, uint32_t tiles16, uint32_t rows, uint32_t B,
                               const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ csr,
                               const uint16_t* __restrict__ x, uint32_t x_stride,
                               const uint16_t* __restrict__ xT, void* y, uint32_t y_stride,
                               int y_f16, int with_dense, int with_csr) {
    constexpr uint32_t P = 32 / XB;
    pdl_trigger();
    pdl_wait();  // the segments of the preceding bstream_gemv
    const uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31, b = lane % XB, k = lane / XB;
    if (r >= rows) return;  // whole warps
    const uint32_t q16 = r >> 4, rr = r & 15u;
    uint32_t sb = 0, rp = 0;
    if (with_dense && lane < 2 * phases) sb = seg_base[(lane >> 1) * tiles16 + q16 + (lane & 1)];
    if (with_csr && lane >= 30) rp = row_ptr[r + (lane - 30)];
    float s = 0.f;
    if (with_dense) {
        for (uint32_t ph = 0; ph < phases; ++ph) {
            uint32_t s0, s1;
            if (phases <= 16) {
                s0 = __shfl_sync(0xffffffffu, sb, 2 * ph);
                s1 = __shfl_sync(0xffffffffu, sb, 2 * ph + 1);
            } else {
                s0 = seg_base[ph * tiles16 + q16];
                s1 = seg_base[ph * tiles16 + q16 + 1];
            }
#pragma unroll 4
            for (uint32_t sg = s0 + k; sg < s1; sg += P) s += __ldcg(part + (size_t(sg) * 16 + rr) * XB + b);
        }
    }
    if (with_csr) {
        const uint32_t q0 = __shfl_sync(0xffffffffu, rp, 30), q1 = __shfl_sync(0xffffffffu, rp, 31);
        const bool live = b < B;
        const uint16_t* xb = xT ? xT + (live ? b : 0u) : x + size_t(live ? b : 0u) * x_stride;
        const uint32_t xs = xT ? uint32_t(XB) : 1u;
        constexpr uint32_t U = 32 / P;  // entries per lane per round of 32
        float c = 0.f;
        // rounds of 32 entries: one coalesced load (an entry per lane), then
        // part k gathers x for entries k, k + P, .. -- all in flight together
        for (uint32_t base = q0; base < q1; base += 32) {
            const uint32_t n = min(32u, q1 - base);
            const uint32_t ent = lane < n ? __ldg(csr + base + lane) : 0u;
            uint32_t ev[U];
            uint16_t xv[U];
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                const uint32_t j = u * P + k;
                ev[u] = __shfl_sync(0xffffffffu, ent, j);
                xv[u] = live && j < n ? ld_cg_u16(xb + size_t(ev[u] & 0xffffu) * xs) : uint16_t(0);
            }
#pragma unroll
            for (uint32_t u = 0; u < U; ++u)
                if (live && u * P + k < n) c = fma_h(uint16_t(ev[u] >> 16), xv[u], c);
        }
        s += c;
    }
#pragma unroll
    for (uint32_t o = XB; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (k != 0 || b >= B) return;
    if (y_f16)
        static_cast<__half*>(y)[size_t(b) * y_stride + r] = __float2half_rn(s);
    else
        static_cast<float*>(y)[size_t(b) * y_stride + r] = s;
}

template <class K, class... A>
static cudaError_t launch_pdl_bs(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ---- host plan -------------------------------------------------------------


// Split a layer (tiles4 4-row tiles, ns spans) for B <= 8 * nb vectors over
// `grid` CTAs.  Pure host arithmetic (unit-tested through the C ABI).
BStreamPlanHost bstream_plan(uint32_t tiles4, uint32_t ns, uint32_t bits, uint32_t nb,
                             uint32_t grid, uint32_t warps) {
    BStreamPlanHost pl;
    const uint32_t kBsWarps = warps == 16 ? 16u : 8u;
    pl.warps = kBsWarps;
    const uint32_t T = (tiles4 + 3) / 4;
    const uint32_t smax = nb == 2 ? 8u : 16u;  // 64 KB of staged x per phase
    const uint32_t P = std::max<uint32_t>(1, (ns + smax - 1) / smax);  // <= 255 (wdesc .w)
    pl.phases = P;
    pl.phase_span.resize(P + 1);
    for (uint32_t k = 0; k <= P; ++k) pl.phase_span[k] = uint32_t(uint64_t(k) * ns / P);
    for (uint32_t k = 0; k < P; ++k)
        pl.max_span = std::max(pl.max_span, pl.phase_span[k + 1] - pl.phase_span[k]);
    pl.cs = kBsWarps == 16 ? 2u : bits == 3 ? 4u : 3u;
    grid = std::max(grid, P);
    pl.grid = grid;
    // CTAs per phase in proportion to the phase's spans (>= 1 each)
    std::vector<uint32_t> gp(P);
    uint32_t used = 0;
    for (uint32_t k = 0; k < P; ++k) {
        const uint32_t sp = pl.phase_span[k + 1] - pl.phase_span[k];
        gp[k] = std::max<uint32_t>(1, uint32_t(uint64_t(grid) * sp / ns));
        used += gp[k];
    }
    // floor(grid * sp / ns) >= 1 for balanced phases, so used <= grid here
    for (uint32_t k = 0; used < grid; k = (k + 1) % P, ++used) ++gp[k];
    pl.cta_pre.assign(P + 1, 0);
    for (uint32_t k = 0; k < P; ++k) pl.cta_pre[k + 1] = pl.cta_pre[k] + gp[k];
    // warp ranges (bs_warp_range: the kernel's own arithmetic), then segment
    // counts per (phase, tile16)
    pl.wdesc.assign(size_t(grid) * kBsWarps * 4, 0);
    std::vector<uint32_t> pieces(size_t(P) * T, 0);
    for (uint32_t cta = 0; cta < grid; ++cta)
        for (uint32_t w = 0; w < uint32_t(kBsWarps); ++w) {
            uint32_t k, a, g, wb, we;
            bs_warp_range(pl.phase_span.data(), pl.cta_pre.data(), P, T, cta, w, kBsWarps, &k, &a, &g,
                          &wb, &we);
            const uint32_t S = pl.phase_span[k + 1] - pl.phase_span[k];
            uint32_t* d = &pl.wdesc[(size_t(cta) * kBsWarps + w) * 4];
            d[0] = wb;
            d[1] = we;
            d[3] = bs_pack_w(k, a, g);
            if (wb < we)
                for (uint32_t q = wb / S; q <= (we - 1) / S; ++q) ++pieces[size_t(k) * T + q];
        }
    pl.seg_base.assign(size_t(P) * T + 1, 0);
    for (size_t z = 0; z < size_t(P) * T; ++z) pl.seg_base[z + 1] = pl.seg_base[z] + pieces[z];
    pl.nseg = pl.seg_base[size_t(P) * T];
    // each warp's first segment: seg_base of its first tile + the earlier warps on that tile
    std::vector<uint32_t> seen(size_t(P) * T, 0);
    for (uint32_t c = 0; c < grid; ++c)
        for (uint32_t w = 0; w < uint32_t(kBsWarps); ++w) {
            uint32_t* d = &pl.wdesc[(size_t(c) * kBsWarps + w) * 4];
            const uint32_t k = d[3] & 0xffu;
            const uint32_t S = pl.phase_span[k + 1] - pl.phase_span[k];
            if (d[0] >= d[1]) continue;
            const uint32_t q0 = d[0] / S, q1 = (d[1] - 1) / S;
            d[2] = pl.seg_base[size_t(k) * T + q0] + seen[size_t(k) * T + q0];
            for (uint32_t q = q0; q <= q1; ++q) ++seen[size_t(k) * T + q];
        }
    return pl;
}

size_t bstream_smem_bytes(uint32_t bits, uint32_t nb, uint32_t max_span, uint32_t cs,
                          uint32_t warps) {
    const uint32_t kBsWarps = warps, kBsSlots = bs_slots(warps);
    const uint32_t LW = bits == 3 ? 4u : 8u, UW = bits * 32u;
    const size_t slot = 2u * (cs * UW + 16u) + 2u * cs * UW + 16u * LW;  // BStreamParams
    return kBsBarBytes + size_t(kBsWarps) * kBsSlots * slot * 4 +
           size_t(8 * nb) * (max_span * kSpanCols + 32) * 2;
}


// mode: 0 LUT part, 1 CSR part, 2 fused
cudaError_t launch_bstream(uint32_t bits, uint32_t nb, const BStreamDevPlan& pl, const uint32_t* idx,
                           const uint32_t* lut, const uint32_t* row_ptr, const uint32_t* csr,
                           uint32_t rows, uint32_t cols, uint32_t ns, uint32_t tiles4,
                           const uint16_t* x, uint32_t x_stride, uint32_t B, void* y,
                           uint32_t y_stride, bool y_f16, int mode, cudaStream_t st) {
    const int with_dense = mode != 1, with_csr = mode != 0;
    const uint16_t* xT = with_dense && with_csr ? pl.xT : nullptr;
    if (with_dense) {
        BStreamParams p{};
        p.idx = idx;
        p.lut = lut;
        p.x = x;
        p.part = pl.part;
        p.xT = const_cast<uint16_t*>(xT);
        p.wdesc = pl.wdesc;
        p.seg_base = pl.seg_base;
        p.phases = pl.phases;
        for (uint32_t k = 0; k <= pl.phases; ++k) {
            p.phase_span[k] = pl.phase_span_h[k];
            p.cta_pre[k] = pl.cta_pre_h[k];
        }
        p.cols = cols;
        p.ns = ns;
        p.tiles4 = tiles4;
        p.tiles16 = pl.tiles16;
        p.B = B;
        p.x_stride = x_stride;
        p.xs_stride = pl.max_span * kSpanCols + 32;  // 32 mod 64 halves: conflict-free LDS.128
        p.cs = pl.cs;
        const uint32_t UW = bits * 32u, LW = bits == 3 ? 4u : 8u;
        p.pw = pl.cs * UW + 16u;
        p.lut_off = p.pw + pl.cs * UW;
        p.pair = p.lut_off + 16u * LW;
        p.slot_words = p.pair + p.pw + pl.cs * UW;
        const size_t smem = bstream_smem_bytes(bits, nb, pl.max_span, pl.cs, pl.warps);
        using K = void (*)(BStreamParams);
        static const K kerns[8] = {bstream_gemv<3, 1, 8>,  bstream_gemv<3, 2, 8>,
                                   bstream_gemv<4, 1, 8>,  bstream_gemv<4, 2, 8>,
                                   bstream_gemv<3, 1, 16>, bstream_gemv<3, 2, 16>,
                                   bstream_gemv<4, 1, 16>, bstream_gemv<4, 2, 16>};
        const int ki = (pl.warps == 16 ? 4 : 0) + (bits == 3 ? 0 : 2) + (nb == 2 ? 1 : 0);
        const K k = kerns[ki];
        // the shared-memory opt-in once per kernel and device (the attribute
        // call costs microseconds of host time per product otherwise)
        static bool attr_done[8][64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        cudaError_t e = cudaSuccess;
        if (dev < 0 || dev >= 64 || !attr_done[ki][dev]) {
            int max_optin = 0;
            cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            if (size_t(max_optin) < smem) return cudaErrorInvalidValue;
            e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin);
            if (e != cudaSuccess) return e;
            if (dev >= 0 && dev < 64) attr_done[ki][dev] = true;
        }
        if ((e = launch_pdl_bs(k, dim3(pl.grid), dim3(pl.warps * 32), smem, st, p)) != cudaSuccess)
            return e;
    }
    const dim3 fg((rows + 7) / 8);  // one warp per row
    return nb == 2 ? launch_pdl_bs(bstream_finish<16>, fg, dim3(256), 0, st, pl.part, pl.seg_base,
                                   pl.phases, pl.tiles16, rows, B, row_ptr, csr, x, x_stride, xT, y,
                                   y_stride, y_f16 ? 1 : 0, with_dense, with_csr)
                   : launch_pdl_bs(bstream_finish<8>, fg, dim3(256), 0, st, pl.part, pl.seg_base,
                                   pl.phases, pl.tiles16, rows, B, row_ptr, csr, x, x_stride, xT, y,
                                   y_stride, y_f16 ? 1 : 0, with_dense, with_csr);
}

}  // namespace sqz
